"""Device verify (sgx_verify_solutions) vs the reference's cmd_verify checks
(oracle restatement over eval_cnf / SolutionSet, one host thread) on the
solution text of a sampler run."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import RefInstance  # noqa: E402
from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig,  # noqa: E402
                                   load_instance, write_dimacs)

for name, batch, restarts in [("c2_iscas", 65536, 0), ("c3a_or50", 1 << 20, 0), ("c4_blasted", 32768, 0)]:
    inst = load_instance(name)
    dc = DeviceCircuit.from_instance(inst)
    s = Sampler(dc, SamplerConfig(batch=batch, iterations=5, seed=1))
    st = s.run()
    text = s.format_solutions()
    s.close()
    dc.verify_solutions(text[: 1 << 20].rsplit(b"\n", 1)[0] + b"\n")  # warm
    t = time.perf_counter()
    got = dc.verify_solutions(text)
    dt = time.perf_counter() - t
    ref = RefInstance.from_dimacs(write_dimacs(inst.cnf))
    # the reference on a bounded prefix (it runs ~1e5x slower): scale by bytes
    cut = text[: min(len(text), 64 << 20)].rsplit(b"\n", 1)[0] + b"\n"
    want = ref.verify_text(cut)
    same = ref.verify_text(text[: 1 << 20].rsplit(b"\n", 1)[0] + b"\n")["kind"] == \
        dc.verify_solutions(text[: 1 << 20].rsplit(b"\n", 1)[0] + b"\n")["kind"]
    ref_rate = len(cut) / want["wall_s"]
    print(f"{name:11s} {got['checked']:9d} solutions {len(text) / 1e9:7.3f} GB text: device verify {dt * 1e3:8.1f} ms "
          f"({len(text) / dt / 1e9:6.2f} GB/s, ok={got['ok']})   reference {want['checked']} solutions in "
          f"{want['wall_s']:7.2f} s ({ref_rate / 1e6:7.2f} MB/s)  x{(len(text) / dt) / ref_rate:8.1f}  "
          f"same_verdict={same}", flush=True)
    dc.close()
