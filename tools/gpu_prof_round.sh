# Round profile set: launch lists (C2, C3a, C4) and one ncu --set full capture of the C2 top kernels.
for W in c2_iscas c3a_or50 c4_blasted; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline --no-ttk > /dev/null 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_backward|k_forward|k_harvest" -c 4 -o gpurun_out/prof_c2_round python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-ttk > /dev/null 2>&1
ls gpurun_out
