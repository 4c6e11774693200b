import os, sys; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import glob, os, time, numpy as np, sys
from paper_2502_08673_b200 import load_instance, extract_circuit
from paper_2502_08673_b200.circuit import DATA_DIR
names = [os.path.basename(p)[:-7] for p in sorted(glob.glob(DATA_DIR + "/*.cnf.gz"))]
names += ["c5/" + os.path.basename(p)[:-7] for p in sorted(glob.glob(DATA_DIR + "/c5/*.cnf.gz"))]
bad = 0
for n in names:
    inst = load_instance(n)
    t = time.perf_counter(); r = extract_circuit(inst.cnf); dt = time.perf_counter() - t
    c, g = r.circuit, inst.circuit
    ok = all(np.array_equal(getattr(c, f), getattr(g, f)) for f in ("kind", "a", "b", "var", "inputs", "out_var", "out_tgt"))
    ok = ok and r.unsat == inst.unsat and r.unsat_note == inst.unsat_note
    if not ok:
        bad += 1
        print("MISMATCH", n, c.n_nodes, g.n_nodes, len(c.inputs), len(g.inputs), len(c.out_var), len(g.out_var), r.unsat, inst.unsat, r.unsat_note, "|", inst.unsat_note)
    elif n.startswith("c") and not n.startswith("c5"): print("ok", n, c.n_nodes, f"{dt*1e3:.1f} ms")
print("bad", bad, "of", len(names))
