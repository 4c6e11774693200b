timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/kit_pytest.txt 2>&1; tail -2 gpurun_out/kit_pytest.txt
timeout 300 python tools/ttk_trace.py 2>&1 | tail -6
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/kit_bench.json 2>/dev/null; python -c "
import json; d=json.loads([l for l in open('gpurun_out/kit_bench.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['time_to_1k'])"
