"""Native extraction (csrc/sgx_extract.cpp) vs the reference's extract + build
on the same CNFs, one host thread each; checks the circuits are identical."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle.oracle import RefInstance, RefLib  # noqa: E402
from paper_2502_08673_b200 import extract_circuit, load_instance, write_dimacs  # noqa: E402

names = sys.argv[1:] or ["c1a_planted3sat", "c2_iscas", "c3b_or100", "c4_blasted"]
R = RefLib()
for n in names:
    inst = load_instance(n)
    text = write_dimacs(inst.cnf)
    te, tb = R.extract_seconds(text, 1)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        r = extract_circuit(inst.cnf)
        best = min(best, time.perf_counter() - t)
    ref = RefInstance.from_dimacs(text)
    same = all(np.array_equal(getattr(r.circuit, f), getattr(ref, f))
               for f in ("kind", "a", "b", "var", "inputs", "out_var", "out_tgt"))
    print(f"{n:18s} clauses {inst.cnf.n_clauses:7d} nodes {r.circuit.n_nodes:7d}  reference "
          f"extract {te * 1e3:8.1f} ms + build {tb * 1e3:6.1f} ms   native {best * 1e3:7.1f} ms  "
          f"x{(te + tb) / best:5.1f}  identical={same}")
