# Round-end validation: GPU tests, smoke, the default bench line, status table, profiles.
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/final_pytest_gpu.txt 2>&1; tail -2 gpurun_out/final_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final_smoke.txt 2>&1; tail -1 gpurun_out/final_smoke.txt
timeout 600 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; tail -c 1500 gpurun_out/final_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final_bench_ref.json 2>&1; tail -c 600 gpurun_out/final_bench_ref.json
bash tools/gpu_status.sh
bash tools/gpu_prof_round.sh
python tools/extract_bench.py > gpurun_out/final_extract.txt 2>&1; cat gpurun_out/final_extract.txt
