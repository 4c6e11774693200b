"""Per-row restart (RestartPolicy.REINIT_ROWS) against the whole-batch policy:
unique valid solutions and device time at the same steps, per workload."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig,  # noqa: E402
                                   load_instance)

CASES = [("c2_iscas", 65536, 10), ("c4_blasted", 65536, 10), ("c3a_or50", 1 << 20, 10), ("mux_chain14", 65536, 10)]
for name, batch, restarts in CASES:
    dc = DeviceCircuit.from_instance(load_instance(name))
    out = []
    for pol in (RestartPolicy.REINIT_ON_EXHAUST, RestartPolicy.REINIT_ROWS):
        cfg = SamplerConfig(batch=batch, iterations=5, seed=1, restart=pol, max_restarts=restarts,
                            solution_capacity=(restarts + 2) * 6 * batch)
        s = Sampler(dc, cfg)
        s.run()  # warm
        st = s.run()
        out.append((pol.name, st.unique_count, st.device_ms))
        s.close()
    dc.close()
    (n0, u0, t0), (n1, u1, t1) = out
    print(f"{name:12s} batch {batch:8d}  whole-batch {u0:10d} in {t0:8.2f} ms ({u0 / t0 * 1e3:12.0f}/s)   "
          f"per-row {u1:10d} in {t1:8.2f} ms ({u1 / t1 * 1e3:12.0f}/s)   unique x{u1 / max(1, u0):.3f} "
          f"rate x{(u1 / t1) / max(1e-9, u0 / t0):.3f}", flush=True)
