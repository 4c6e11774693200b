for W in c3a_or50 c3b_or100 c4_blasted; do
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline --no-ttk > /dev/null 2>&1
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/bench_$W.txt 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_backward|k_forward|k_harvest" -c 3 -o gpurun_out/prof_c4 python bench.py --workload c4_blasted --steps 1 --warmup 0 --no-cpu-baseline --no-ttk > /dev/null 2>&1
