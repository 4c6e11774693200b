"""How much of the soft tape is exactly 0 or 1 as GD proceeds (sizing a
possible exact row compression): C4 / C2 at 4,096 rows, V from the
sampler after k steps, the forward tape in the reference layout [node][batch]
through the parity tap (sgx_forward), then the fraction of values in {0, 1}
and of 128-sample rows made only of them (the unit a compressed row would
cover)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2502_08673_b200 import DeviceCircuit, Sampler, SamplerConfig, load_instance  # noqa: E402
from paper_2502_08673_b200 import autodiff as AD  # noqa: E402

for name in sys.argv[1:] or ["c4_blasted", "c2_iscas"]:
    inst = load_instance(name)
    dc = DeviceCircuit.from_instance(inst)
    s = Sampler(dc, SamplerConfig(batch=4096, iterations=5, seed=1))
    s.init(0)
    for k in range(6):
        v = s.logits()
        p = AD.embed(v)
        tape, _ = AD.forward(dc, p)  # [node][batch]
        t = tape.reshape(tape.shape[0], -1, 128)
        exact = (t == 0.0) | (t == 1.0)
        rows = exact.all(axis=2)
        print(f"{name} step {k}: values in {{0,1}} {exact.mean():.3f}; 128-sample rows all in {{0,1}} {rows.mean():.3f}",
              flush=True)
        s.step()
    s.close()
    dc.close()
