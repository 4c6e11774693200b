# A/B: alternate library builds (libsatgrad_b200_<tag>.so) on the bench
set -x
cp paper_2502_08673_b200/libsatgrad_b200.so /tmp/main.so
for tag in ${TAGS}; do
  cp paper_2502_08673_b200/libsatgrad_b200_$tag.so paper_2502_08673_b200/libsatgrad_b200.so
  timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_$tag.txt 2>&1
done
cp /tmp/main.so paper_2502_08673_b200/libsatgrad_b200.so
for env in ${ENVS}; do env $env timeout 300 python bench.py --steps 5 --warmup 2 --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_env_$env.txt 2>&1; done
