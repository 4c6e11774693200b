# live harvest vs the full-tape shared-memory / global harvests on C2, C3a, C4
for W in c2_iscas c3a_or50 c4_blasted; do
  for H in live smem g; do
    e=""; [ "$H" != live ] && e="SGX_HARVEST=$H"
    env $e timeout 300 python bench.py --workload $W --steps 3 --warmup 2 --no-cpu-baseline --no-ttk > gpurun_out/hab_${W}_$H.txt 2>&1
  done
done
python tools/summ.py "gpurun_out/hab_*.txt"
