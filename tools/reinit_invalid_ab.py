"""Restart policies against each other on the bench workloads: unique valid
solutions per device second for REINIT_ON_EXHAUST (the reference's), REINIT_ROWS
and REINIT_INVALID at several reinit_age values, same restarts."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig,  # noqa: E402
                                   load_instance)

CASES = [("c2_iscas", 65536, 10), ("c4_blasted", 65536, 6), ("c3a_or50", 1 << 20, 10)]
VARIANTS = [(RestartPolicy.REINIT_ON_EXHAUST, 0), (RestartPolicy.REINIT_ROWS, 0)] + \
           [(RestartPolicy.REINIT_INVALID, a) for a in (1, 2, 3, 4)]
for name, batch, restarts in CASES:
    dc = DeviceCircuit.from_instance(load_instance(name))
    base = None
    for pol, age in VARIANTS:
        cfg = SamplerConfig(batch=batch, iterations=5, seed=1, restart=pol, max_restarts=restarts,
                            reinit_age=age, solution_capacity=(restarts + 2) * 6 * batch)
        s = Sampler(dc, cfg)
        s.run()  # warm
        st = s.run()
        s.close()
        rate = st.unique_count / st.device_ms * 1e3
        base = base or rate
        print(f"{name:12s} {pol.name:18s} age {age}  unique {st.unique_count:10d}  attempts {st.attempts:11d}  "
              f"{st.device_ms:9.2f} ms  {rate:13.0f}/s  x{rate / base:.3f}", flush=True)
    dc.close()
