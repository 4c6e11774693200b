# Upper bound of barrier removal on the staged backward (results deliberately wrong): ncu backward time + DRAM bytes
cp paper_2502_08673_b200/libsatgrad_b200.so /tmp/main.so
for tag in main nb w8 w8nb w16 w16nb; do
  if [ $tag = main ]; then cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so; else cp paper_2502_08673_b200/libsatgrad_b200_$tag.so paper_2502_08673_b200/libsatgrad_b200.so; fi
  SGX_BWD=async timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_backward -c 2 --csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ttk > gpurun_out/nobar_$tag.csv 2>/dev/null
done
cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
python tools/traffic_summ.py "gpurun_out/nobar_*.csv"
