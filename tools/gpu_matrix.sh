# A/B matrix: each CASES entry is TAG:ENV (TAG = library variant suffix or "main",
# ENV = comma-separated VAR=VALUE list or "-").  Prints one summary line per case.
cp paper_2502_08673_b200/libsatgrad_b200.so /tmp/main.so
for c in ${CASES}; do
  tag=${c%%:*}; envs=${c#*:}
  if [ "$tag" = main ]; then cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so;
  else cp paper_2502_08673_b200/libsatgrad_b200_$tag.so paper_2502_08673_b200/libsatgrad_b200.so; fi
  e=""; [ "$envs" != "-" ] && e=$(echo "$envs" | tr ',' ' ')
  env $e timeout 300 python bench.py --steps ${STEPS:-5} --warmup 3 --no-cpu-baseline --no-ttk ${BENCH_ARGS} > "gpurun_out/bench_m_${tag}_${envs}.txt" 2>&1
done
cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
python tools/summ.py "gpurun_out/bench_m_*.txt"
