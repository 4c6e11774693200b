"""Small runs of the per-row restart kernels (k_reinit_mask, k_reinit_rows) for
compute-sanitizer: REINIT_ROWS / REINIT_INVALID at once and lagged
(SGX_REINIT_LAG=1), and the default forward-only harvest overlap."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import RestartPolicy, SamplerConfig, load_instance, run_instance  # noqa: E402

for lag in ("0", "1"):
    os.environ["SGX_REINIT_LAG"] = lag
    for name, b in (("c2_iscas", 2048), ("c3a_or50", 4096), ("c4_blasted", 256)):
        inst = load_instance(name)
        for pol in (RestartPolicy.REINIT_ROWS, RestartPolicy.REINIT_INVALID):
            res = run_instance(inst, SamplerConfig(batch=b, iterations=3, seed=1, restart=pol, max_restarts=1,
                                                   reinit_age=1))
            print(name, pol.name, "lag", lag, res.stats.unique_count, flush=True)
