# quick loop: GPU parity subset + bench + launch list
set -x
timeout 600 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps ${STEPS:-5} --warmup 2 ${BENCH_ARGS} > gpurun_out/bench1.txt 2>&1; echo "bench rc=$?" >> gpurun_out/bench1.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_launch_run.txt 2>&1
if [ -n "$NCU_FULL" ]; then timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_FULL" -c ${NCU_COUNT:-2} -o gpurun_out/prof_q python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_full_run.txt 2>&1; fi
tail -4 gpurun_out/pytest_gpu.txt; tail -2 gpurun_out/bench1.txt
