"""Backward pass schedules in the row-granular L2 model (tools/l2sim.py):
ALAP (the layout's), ASAP, and a local search that moves every node inside
its slack window (after all consumers, before all operands) to the pass where
most of the rows it touches are touched within +-W passes.  Design aid for
DESIGN.md section 7; prints modelled backward DRAM (read, write, total) GB.

usage: python tools/bwd_sched.py INSTANCE [W] [ITERS]
"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.pop("L2SIM_SPLIT", None)
import numpy as np
from collections import defaultdict
import l2sim

name = sys.argv[1] if len(sys.argv) > 1 else "c4_blasted"
P = l2sim.program(name, "alap")
real, lv, cons = P["real"], P["lv"].copy(), P["cons"]
N = P["N"]; a, b, base = P["a"], P["b"], P["base"]
rows = [n for n in range(N) if real[n]]
# operands (materialized) of each real node
opsof = {n: [base[o] for o in (a[n], b[n]) if o >= 0] for n in rows}
def sim(blv, tiles=512):
    Q = dict(P); Q["lv"] = blv
    rd, wr = l2sim.simulate(Q, tiles, 110.0, True, True, False)
    return rd, wr, rd + wr
print("alap", sim(lv))
# asap
asap = np.zeros(N, int)
for n in rows:
    asap[n] = 1 + max([asap[o] for o in opsof[n]], default=-1)
print("asap", sim(asap))
W = int(sys.argv[2]) if len(sys.argv) > 2 else 1
def accesses(n):
    acc = [("a", n)] if (cons[n] or P["kind"][n] == 0) else []
    for (cn, other) in cons[n]:
        acc.append(("a", cn))
        if other >= 0: acc.append(("t", other))
    if n in P["outs"]: acc.append(("t", n))
    return acc
bl = lv.copy()
where = defaultdict(lambda: defaultdict(int))  # key -> pass -> count
for n in rows:
    for k in accesses(n): where[k][bl[n]] += 1
# adjoint writes of consumers are accesses at the consumer's pass (already added as ("a", n) of the consumer)
t0 = time.time()
for it in range(int(sys.argv[3]) if len(sys.argv) > 3 else 2):
    moved = 0
    for n in sorted(rows, key=lambda n: -bl[n]):
        hi = min([bl[c] for (c, _) in cons[n]], default=P["L"] + 1) - 1
        lo = max([bl[o] for o in opsof[n]], default=-1) + 1
        if lo >= hi: continue
        acc = accesses(n)
        for k in acc:
            where[k][bl[n]] -= 1
        cands = {bl[n]}
        for k in acc:
            for p in where[k]:
                if where[k][p] > 0:
                    for q in range(p - W, p + W + 1):
                        if lo <= q <= hi: cands.add(q)
        def score(p):
            s = 0
            for k in acc:
                d = where[k]
                if any(d.get(q, 0) > 0 for q in range(p - W, p + W + 1)): s += 1
            return s
        best = max(sorted(cands, key=lambda p: -p), key=score)  # ties -> highest pass (ALAP-like)
        if score(best) <= score(bl[n]): best = bl[n]
        if best != bl[n]: moved += 1
        bl[n] = best
        for k in acc:
            where[k][bl[n]] += 1
    print("iter", it, "moved", moved, sim(bl), f"{time.time()-t0:.1f}s", flush=True)

