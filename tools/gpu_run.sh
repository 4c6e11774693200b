# Parameterised GPU-box runner: bash tools/gpu_run.sh "<cmd1>" "<cmd2>" ...
# Each command runs under a 20 min timeout; output lands in gpurun_out/run_<i>.txt
# and its tail is echoed (gpurun only returns the tail of stdout).
set -u
mkdir -p gpurun_out
i=0
for c in "$@"; do
  i=$((i+1))
  echo "== [$i] $c"
  timeout ${GPU_STEP_TIMEOUT:-1200} bash -c "$c" > gpurun_out/run_$i.txt 2>&1
  echo "rc=$?"
  tail -${GPU_TAIL:-25} gpurun_out/run_$i.txt | cut -c1-400
done
