# A/B: 8 warps per tile (-DSGX_WARPS=8) against the default 4, C2 / C3a / C4, alternating.
cp paper_2502_08673_b200/libsatgrad_b200.so /tmp/main.so
for W in c2_iscas c4_blasted c3a_or50; do
  for rep in 1 2; do
    for tag in main w8; do
      [ $tag = w8 ] && cp paper_2502_08673_b200/libsatgrad_b200_w8.so paper_2502_08673_b200/libsatgrad_b200.so || cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
      timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-ttk > gpurun_out/w8_${W}_${tag}_$rep.txt 2>&1
    done
  done
done
cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
python tools/summ.py "gpurun_out/w8_*.txt"
