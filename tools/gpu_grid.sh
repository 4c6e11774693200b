# persistent-grid sweep for the soft kernels (forward / backward)
for g in ${GRIDS:-0 148 296 444}; do
  SGX_GRID_FWD=$g SGX_GRID_BWD=$g timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-ttk ${BENCH_ARGS} > gpurun_out/bench_grid_$g.txt 2>&1
  python -c "
import json
l=[x for x in open('gpurun_out/bench_grid_$g.txt') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('grid $g', d and (round(d['value']), d.get('phase_ms')))
"
done
