"""compute-sanitizer cases for the per-row restart, the device verifier and
the device formatter (small sizes)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig,  # noqa: E402
                                   load_instance, verify_solutions)
for name, b in (("c1b_random", 1024), ("c3a_or50", 4096), ("c2_iscas", 512)):
    inst = load_instance(name)
    dc = DeviceCircuit.from_instance(inst)
    s = Sampler(dc, SamplerConfig(batch=b, iterations=2, seed=1, restart=RestartPolicy.REINIT_ROWS,
                                  max_restarts=1))
    st = s.run()
    text = s.format_solutions()
    v = dc.verify_solutions(text)
    lines = text.split(b"\n")
    bad = b"\n".join(lines[:3] + [lines[1]] + lines[3:])  # a duplicate
    w = verify_solutions(inst.cnf, bad)
    print(name, st.unique_count, v["ok"], w["kind"], flush=True)
    s.close()
    dc.close()
