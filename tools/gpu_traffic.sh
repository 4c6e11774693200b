# DRAM bytes / duration of the soft kernels per variant: CASES as in gpu_matrix.sh
cp paper_2502_08673_b200/libsatgrad_b200.so /tmp/main.so
for c in ${CASES}; do
  tag=${c%%:*}; envs=${c#*:}
  if [ "$tag" = main ]; then cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so;
  else cp paper_2502_08673_b200/libsatgrad_b200_$tag.so paper_2502_08673_b200/libsatgrad_b200.so; fi
  e=""; [ "$envs" != "-" ] && e=$(echo "$envs" | tr ',' ' ')
  env $e timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct \
    --clock-control none -k regex:"${NCU_K:-k_backward|k_forward}" -c ${NCU_COUNT:-4} --csv \
    python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ttk ${BENCH_ARGS} > "gpurun_out/traffic_${tag}_${envs}.csv" 2>/dev/null
done
cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
python tools/traffic_summ.py "gpurun_out/traffic_*.csv"
