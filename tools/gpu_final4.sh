timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final4_pytest_gpu.txt 2>&1; tail -3 gpurun_out/final4_pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 --no-ttk > gpurun_out/final4_bench.json 2>/dev/null; python -c "
import json; d=json.loads([l for l in open('gpurun_out/final4_bench.json') if l.startswith('{')][-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['clocks'], d['gpu_launches'])"
