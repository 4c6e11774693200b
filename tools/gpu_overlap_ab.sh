for W in c3a_or50 c3b_or100 c2_iscas; do
  for O in 1 0; do for rep in 1 2; do
    SGX_OVERLAP=$O timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-ttk > gpurun_out/ov_${W}_${O}_$rep.txt 2>&1
  done; done
done
for f in gpurun_out/ov_*.txt; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', round(d['value']/1e6,1), 'M/s', round(d['device_s']*1000,1), 'ms', d['phase_ms'])"; done
