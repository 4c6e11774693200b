# A/B: forward with group records one group ahead (current) vs the previous build (prev).
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "forward or golden or trajectory or c5" > gpurun_out/fab_pytest.txt 2>&1; tail -2 gpurun_out/fab_pytest.txt
cp paper_2502_08673_b200/libsatgrad_b200.so /tmp/main.so
for W in c2_iscas c4_blasted c3a_or50; do
  for rep in 1 2; do
    for tag in prev main; do
      [ $tag = prev ] && cp paper_2502_08673_b200/libsatgrad_b200_prev.so paper_2502_08673_b200/libsatgrad_b200.so || cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
      timeout 300 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-ttk > gpurun_out/fab_${W}_${tag}_$rep.txt 2>&1
    done
  done
done
cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
python tools/summ.py "gpurun_out/fab_*.txt"
