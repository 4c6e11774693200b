# launch list + one ncu --set full capture of the soft kernels and the harvest
W=${WORKLOAD:-c2_iscas}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W.csv python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline --no-ttk > gpurun_out/ncu_launch_run.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${NCU_K:-k_backward|k_forward|k_harvest_smem}" -c ${NCU_COUNT:-3} -o gpurun_out/prof_$W python bench.py --workload $W --steps 1 --warmup 0 --no-cpu-baseline --no-ttk > gpurun_out/ncu_full_run.txt 2>&1
ls -la gpurun_out
