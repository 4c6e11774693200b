#!/bin/bash
# A/B runner (GPU box): bench.py over workloads x variants, alternating, then
# a summary (tools/summ.py).  Replaces the round-1 one-off gpu_*.sh scripts.
#
#   bash tools/ab.sh "c4_blasted c2_iscas" "base" "env:SGX_LWPC=2" "so:w8" ...
#
# A variant is "base" (the tree's libsatgrad_b200.so), "env:K=V[,K=V...]"
# (environment knobs: SGX_VEC, SGX_LWPC, SGX_HARVEST, SGX_JIT, SGX_JIT_MINB,
# SGX_PRIO, SGX_OVERLAP, ...), or "so:TAG" (a build from tools/build_variant.sh
# TAG -DFLAG=...).  REPS (default 2) alternations; STEPS / WARMUP for bench.py.
set -u
WL=$1; shift
REPS=${REPS:-2}
mkdir -p gpurun_out
LIB=paper_2502_08673_b200/libsatgrad_b200.so
cp $LIB /tmp/ab_base.so
for W in $WL; do
  for rep in $(seq 1 $REPS); do
    for v in "$@"; do
      cp /tmp/ab_base.so $LIB
      envs=""
      case $v in
        env:*) envs=$(echo ${v#env:} | tr ',' ' ') ;;
        so:*) cp paper_2502_08673_b200/libsatgrad_b200_${v#so:}.so $LIB ;;
      esac
      tag=$(echo "$v" | tr ':=,/' '____')
      env $envs timeout 600 python bench.py --workload $W --steps ${STEPS:-5} --warmup ${WARMUP:-3} \
        --no-cpu-baseline --no-ttk > gpurun_out/bench_ab_${W}_${tag}_$rep.txt 2>&1
    done
  done
done
cp /tmp/ab_base.so $LIB
python tools/summ.py "gpurun_out/bench_ab_*.txt"
