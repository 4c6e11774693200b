set -x
nvidia-smi -L
timeout 240 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
timeout 900 python -m pytest tests -m gpu -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 400 python bench.py --steps ${STEPS:-5} --warmup 2 > gpurun_out/bench1.txt 2>&1; echo "bench rc=$?" >> gpurun_out/bench1.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch_run.txt 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_backward|k_forward|k_bit_eval|k_keys" -c 4 -o gpurun_out/prof_c2 python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_full_run.txt 2>&1
tail -3 gpurun_out/smoke.txt; tail -15 gpurun_out/pytest_gpu.txt; tail -3 gpurun_out/bench1.txt
