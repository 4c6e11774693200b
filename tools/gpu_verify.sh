timeout 900 python -m pytest tests/test_gpu_verify.py -q -x > gpurun_out/verify_pytest.txt 2>&1; tail -15 gpurun_out/verify_pytest.txt
timeout 900 python tools/verify_bench.py 2>&1 | tail -5
