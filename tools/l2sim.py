"""Row-granular L2 model of the soft passes (design aid, not product code).

All concurrent tiles walk the levels in lock-step, so one tape / adjoint row
across T concurrent tiles is one cache block of T*512 B.  LRU over blocks
with optional policies: y (tape) reads inserted cold (evict_first), adjoint
rows discarded after their last read (discard.global.L2: no write-back),
column-input adjoints consumed at their own pass (inline END) instead of an
epilogue.  Reports modelled DRAM GB per backward launch at B samples.

usage: python tools/l2sim.py INSTANCE [--tiles T ...] [--l2 MB]
"""
import argparse
import os
import sys
from collections import OrderedDict

import numpy as np

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2502_08673_b200 import load_instance  # noqa: E402


def program(name, sched="alap"):
    inst = load_instance(name)
    c = inst.circuit
    N, kind, a, b = c.n_nodes, c.kind, c.a, c.b
    cone = np.zeros(N, bool)
    cone[c.out_node] = True
    for n in range(N - 1, -1, -1):
        if cone[n]:
            for o in (a[n], b[n]):
                if o >= 0:
                    cone[o] = True
    real = cone.copy()
    base = np.arange(N)
    for n in range(N):
        if cone[n] and kind[n] in (3, 4) and real[a[n]]:
            real[n] = False
            base[n] = base[a[n]]
    lv = np.zeros(N, int)
    for n in range(N):
        if not real[n]:
            continue
        ops = [base[o] for o in (a[n], b[n]) if o >= 0]
        lv[n] = 1 + max([lv[o] for o in ops], default=-1)
    L = lv[real].max()
    if sched == "alap":
        al = np.full(N, L)
        for n in range(N - 1, -1, -1):
            if not real[n]:
                continue
            for o in (a[n], b[n]):
                if o >= 0:
                    al[base[o]] = min(al[base[o]], al[n] - 1)
        lv = al
    # consumers (materialized) of each real row, through folded nodes
    cons = [[] for _ in range(N)]  # (consumer row, other row)
    for n in range(N):
        if not cone[n] or not real[n]:
            continue
        ops = [o for o in (a[n], b[n]) if o >= 0]
        for i, o in enumerate(ops):
            other = base[ops[1 - i]] if len(ops) == 2 else -1
            cons[base[o]].append((n, other))
    cpi = set(int(x) for x in c.node_of_var[np.asarray(inst.cpi)])
    return dict(N=N, real=real, lv=lv, L=L, cons=cons, kind=kind, a=a, b=b, base=base,
                outs=set(int(x) for x in c.out_node), cpi=cpi)


def simulate(P, tiles, l2_mb=110.0, y_first=False, discard=False, inline_end=False, total_tiles=512):
    blk = tiles * 512
    cap = int(l2_mb * 1e6 // blk)
    lru = OrderedDict()  # key -> dirty
    stats = dict(rd=0, wr=0, rd_t=0, rd_a=0, rd_v=0)

    def evict():
        while len(lru) > cap:
            k, d = lru.popitem(last=False)
            if d:
                stats["wr"] += 1

    def read(k, cold=False):
        if k in lru:
            lru.move_to_end(k)
        else:
            stats["rd"] += 1
            stats["rd_" + k[0]] += 1
            lru[k] = False
            if cold:
                lru.move_to_end(k, last=False)
        evict()

    def write(k):
        lru[k] = True
        lru.move_to_end(k)
        evict()

    real, lv, cons = P["real"], P["lv"], P["cons"]
    rows = [n for n in range(P["N"]) if real[n]]
    by = {}
    for n in rows:
        by.setdefault(lv[n], []).append(n)
    # last pass reading adj[c]
    last = {}
    for n in rows:
        for (cn, other) in cons[n]:
            last[cn] = min(last.get(cn, 1 << 30), lv[n])
    for l in range(P["L"], -1, -1):
        for n in by.get(l, []):
            if n in P["outs"]:
                read(("t", n), cold=y_first)
            for (cn, other) in cons[n]:
                read(("a", cn))
                if other >= 0:
                    read(("t", other), cold=y_first)
            is_in = P["kind"][n] == 0
            if is_in and n in P["cpi"] and inline_end:
                read(("v", n))
                write(("v", n))
            elif cons[n] or is_in:
                write(("a", n))
        if discard:
            for n in by.get(l, []):
                pass
            for cn in [k for k, v in last.items() if v == l]:
                lru.pop(("a", cn), None)
    if not inline_end:
        for n in rows:
            if P["kind"][n] == 0 and n in P["cpi"]:
                read(("a", n))
                read(("v", n))
                write(("v", n))
    for k, d in lru.items():
        if d:
            stats["wr"] += 1
    waves = total_tiles / tiles
    gb = lambda x: x * blk * waves / 1e9
    if os.environ.get("L2SIM_SPLIT"):
        print(f"   reads: tape {gb(stats['rd_t']):.2f} adjoint {gb(stats['rd_a']):.2f} V {gb(stats['rd_v']):.2f} GB")
    return gb(stats["rd"]), gb(stats["wr"])


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("inst")
    ap.add_argument("--tiles", type=int, nargs="*", default=[512, 296, 148])
    ap.add_argument("--l2", type=float, default=110.0)
    ap.add_argument("--sched", default="alap")
    args = ap.parse_args()
    P = program(args.inst, args.sched)
    for t in args.tiles:
        for yf, dc, ie in ([(1, 1, 0)] if os.environ.get("L2SIM_SPLIT") else [(0, 0, 0), (1, 0, 0), (0, 1, 0), (1, 1, 0), (1, 1, 1)]):
            rd, wr = simulate(P, t, args.l2, bool(yf), bool(dc), bool(ie))
            print(f"tiles {t:4d} y_first {yf} discard {dc} inline_end {ie}: rd {rd:.2f} wr {wr:.2f} "
                  f"total {rd + wr:.2f} GB")


def simulate_forward(P, tiles, l2_mb=110.0, total_tiles=512, store_first=False):
    """Forward: per level read operand rows (V columns for inputs), write rows."""
    blk = tiles * 512
    cap = int(l2_mb * 1e6 // blk)
    lru = OrderedDict()
    st = dict(rd=0, wr=0)

    def touch(k, dirty, cold=False):
        if k in lru:
            lru[k] = lru[k] or dirty
            lru.move_to_end(k)
        else:
            if not dirty:
                st["rd"] += 1
            lru[k] = dirty
            if cold:
                lru.move_to_end(k, last=False)
        while len(lru) > cap:
            _, d = lru.popitem(last=False)
            if d:
                st["wr"] += 1

    real, lv = P["real"], P["lv"]
    a, b, base, kind = P["a"], P["b"], P["base"], P["kind"]
    by = {}
    for n in range(P["N"]):
        if real[n]:
            by.setdefault(lv[n], []).append(n)
    for l in range(P["L"] + 1):
        for n in by.get(l, []):
            if kind[n] == 0:
                touch(("v", n), False)
            for o in (a[n], b[n]):
                if o >= 0:
                    touch(("t", base[o]), False)
            touch(("t", n), True, cold=store_first)
    st["wr"] += sum(1 for d in lru.values() if d)
    waves = total_tiles / tiles
    return st["rd"] * blk * waves / 1e9, st["wr"] * blk * waves / 1e9
