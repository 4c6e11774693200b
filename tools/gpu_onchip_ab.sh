for W in c3a_or50 c3b_or100 c2_iscas; do
  for O in 1 0; do
    SGX_ONCHIP=$O timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-ttk 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$W onchip=$O', round(d['value']/1e6,2), 'M/s', round(d['device_s']*1000,1), 'ms', {k: d['phase_ms'][k] for k in ('forward','backward','harvest')})"
  done
done
timeout 900 python -m paper_2502_08673_b200.sweep > gpurun_out/sweep2.txt 2>&1; tail -1 gpurun_out/sweep2.txt | cut -c1-900
