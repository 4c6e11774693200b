"""Run a quota-1000 run_instance n times and exit (interpreter-exit checks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import RestartPolicy, SamplerConfig, load_instance, run_instance  # noqa: E402

name, batch, n = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
inst = load_instance(name)
cfg = SamplerConfig(batch=batch, iterations=5, seed=1, max_solutions=1000, restart=RestartPolicy.REINIT_ON_EXHAUST)
for _ in range(n):
    r = run_instance(inst, cfg)
print("done", r.stats.unique_count, flush=True)
