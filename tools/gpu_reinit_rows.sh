timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "reinit_rows or host_stream or golden" -s > gpurun_out/rr_pytest.txt 2>&1; grep -E "rows .* vs|passed|failed|Error" gpurun_out/rr_pytest.txt | tail -8
timeout 900 python tools/reinit_rows_ab.py 2>&1 | tail -6
