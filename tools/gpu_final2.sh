# Post-change validation: GPU tests, smoke, default bench line.
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/final2_pytest_gpu.txt 2>&1; tail -2 gpurun_out/final2_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/final2_smoke.txt 2>&1; tail -1 gpurun_out/final2_smoke.txt
timeout 600 python bench.py > gpurun_out/final2_bench.json 2> gpurun_out/final2_bench.err; tail -c 700 gpurun_out/final2_bench.json
python tools/extract_bench.py > gpurun_out/final2_extract.txt 2>&1; cat gpurun_out/final2_extract.txt
