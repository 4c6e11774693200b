# Status-table measurements: every workload with its CPU baseline, the C5 sweep.
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/st_c2_iscas.txt 2>&1
for W in c3a_or50 c3b_or100 c4_blasted; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-ttk > gpurun_out/st_$W.txt 2>&1
done
timeout 900 python -m paper_2502_08673_b200.sweep > gpurun_out/st_sweep.txt 2>&1
for f in gpurun_out/st_*.txt; do echo "== $f"; tail -1 $f | cut -c1-400; done
