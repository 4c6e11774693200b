# parity subset then bench at several vector widths
set -x
timeout 600 python -m pytest tests -m gpu -q -x ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for v in ${VECS:-1 2 4}; do
  SGX_VEC=$v timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_v$v.txt 2>&1
done
SGX_VEC=${NCU_VEC:-4} timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_launch_run.txt 2>&1
if [ -n "$NCU_FULL" ]; then SGX_VEC=${NCU_VEC:-4} timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_FULL" -c ${NCU_COUNT:-2} -o gpurun_out/prof_q python bench.py --steps 1 --warmup 0 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/ncu_full_run.txt 2>&1; fi
tail -4 gpurun_out/pytest_gpu.txt
for v in ${VECS:-1 2 4}; do python -c "
import json,sys
l=[x for x in open('gpurun_out/bench_v$v.txt') if x.startswith('{')]
d=json.loads(l[-1]) if l else None
print('vec $v', d and (round(d['value']), d['phase_ms'], round(d['roofline']['frac'],3), d['e2e']['value']))
"; done
