# Final validation: all GPU tests, smoke, the default bench line, the reference arm.
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/final3_pytest_gpu.txt 2>&1; tail -3 gpurun_out/final3_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final3_smoke.txt 2>&1; tail -1 gpurun_out/final3_smoke.txt
timeout 600 python bench.py > gpurun_out/final3_bench.json 2> gpurun_out/final3_bench.err; tail -c 900 gpurun_out/final3_bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/final3_bench_ref.json 2>&1; tail -c 300 gpurun_out/final3_bench_ref.json
