# Live-harvest words per CTA (SGX_LWPC) A/B on C4 and C2.
for W in c4_blasted c2_iscas; do
  for L in 0 1 2 4 8; do
    e=""; [ "$L" != 0 ] && e="SGX_LWPC=$L"
    env $e timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-ttk > gpurun_out/lwpc_${W}_$L.txt 2>&1
  done
done
python tools/summ.py "gpurun_out/lwpc_*.txt"
