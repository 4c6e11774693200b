"""Forward read hints in the row-granular L2 model: a read loads evict_first
when its row is not read again within D levels (SGX_FWD_FAR).  Prints
modelled forward DRAM (read, write) GB per launch at 512 tiles.

usage: python tools/fwd_far_sim.py INSTANCE
"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import l2sim
from collections import OrderedDict
import numpy as np
name = sys.argv[1]
P = l2sim.program(name)
real, lv, a, b, base, kind = P["real"], P["lv"], P["a"], P["b"], P["base"], P["kind"]
N = P["N"]
by = {}
for n in range(N):
    if real[n]: by.setdefault(lv[n], []).append(n)
# read events per row: list of levels
reads = {}
for l in range(P["L"] + 1):
    for n in by.get(l, []):
        for o in (a[n], b[n]):
            if o >= 0: reads.setdefault(base[o], []).append(l)
def sim(tiles, D, l2_mb=110.0, total_tiles=512):
    blk = tiles * 512; cap = int(l2_mb * 1e6 // blk)
    lru = OrderedDict(); st = dict(rd=0, wr=0)
    ptr = {}
    def touch(k, dirty, cold=False):
        if k in lru:
            lru[k] = lru[k] or dirty; lru.move_to_end(k)
        else:
            if not dirty: st["rd"] += 1
            lru[k] = dirty
        if cold: lru.move_to_end(k, last=False)
        while len(lru) > cap:
            _, d = lru.popitem(last=False)
            if d: st["wr"] += 1
    for l in range(P["L"] + 1):
        for n in by.get(l, []):
            if kind[n] == 0: touch(("v", n), False, True)
            for o in (a[n], b[n]):
                if o >= 0:
                    r = base[o]; i = ptr.get(r, 0)
                    rl = reads[r]
                    # advance past reads at this level
                    while i < len(rl) and rl[i] <= l: i += 1
                    ptr[r] = i
                    nxt = rl[i] if i < len(rl) else None
                    cold = nxt is None or (D is not None and nxt - l > D)
                    touch(("t", r), False, cold)
            touch(("t", n), True)
    st["wr"] += sum(1 for d in lru.values() if d)
    w = total_tiles / tiles
    return round(st["rd"] * blk * w / 1e9, 2), round(st["wr"] * blk * w / 1e9, 2)
for D in (None, 16, 32, 48, 64, 96, 128):
    print("D", D, sim(512, D), flush=True)
