"""End-to-end run() timing at C4 bench size, repeated (drain / parked-mapping behaviour with SGX_TRACE=1)."""
import time, sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import load_instance, run_instance, SamplerConfig, RestartPolicy
inst = load_instance("c4_blasted")
steps = int(sys.argv[1])
cfg = SamplerConfig(batch=65536, iterations=5, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=steps - 1)
for k in range(3):
    t = time.perf_counter()
    r = run_instance(inst, cfg, device=0)
    n = r.stats.unique_count
    t1 = time.perf_counter()
    del r
    print(f"run {k}: {n} unique in {t1 - t:.3f} s -> {n / (t1 - t) / 1e6:.2f} M/s; release {time.perf_counter() - t1:.3f} s", flush=True)
