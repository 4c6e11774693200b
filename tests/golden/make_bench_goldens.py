"""Reference goldens at the BENCH batch sizes (VERDICT r1 "next" item 1).

The default kernel selection only kicks in at bench sizes (e.g. the live-slot
harvest ``k_harvest_live`` is chosen once a batch has >= 148 words), so these
runs pin exactly the kernels ``bench.py`` times to the reference's own
``satgrad::run`` (``src/sampler.cpp:89-203``) on the same instance, batch,
seed and iteration budget.

Run in the build container (needs oracle/_ref, i.e. /root/reference):

    make -C oracle ref && python tests/golden/make_bench_goldens.py [name ...]

Writes tests/golden/bench_runs.json: per run the stats, the loss trace, the
per-harvest new-unique trace and the sha256 of the insertion-ordered keys
(the full keys are tens of MB, so only their digest is committed).  Memory:
the reference keeps the whole node-major tape and adjoint ([N][B] f32 each),
C4 at B = 65,536 needs ~47 GB of host RAM.  Results do not depend on the
thread count (autodiff.hpp:10-11), so the runs use every host core.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from make_fixtures import INSTANCES, make  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "bench_runs.json")

# name -> (instance, config).  bench.py's workloads at their bench batch.
BENCH_RUNS = {
    "c3a_2p20_it2": ("c3a_or50", dict(batch=1 << 20, iterations=2, seed=1)),
    "c3b_2p20_it1": ("c3b_or100", dict(batch=1 << 20, iterations=1, seed=1)),
    "c2_65536_it5": ("c2_iscas", dict(batch=65536, iterations=5, seed=1)),
    "c2_65536_quota": ("c2_iscas", dict(batch=65536, iterations=5, seed=3, max_solutions=20000,
                                        restart=True)),
    "c4_65536_it1": ("c4_blasted", dict(batch=65536, iterations=1, seed=1)),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main(names) -> None:
    out = json.load(open(OUT)) if os.path.exists(OUT) else {}
    threads = os.cpu_count() or 1
    for name in names:
        inst_name, cfg = BENCH_RUNS[name]
        gen, param = INSTANCES[inst_name]
        inst = make(gen, param)
        t0 = time.time()
        r = inst.run(use_f32=True, threads=threads, **cfg)
        # Per-harvest slices of the ordered keys: a mismatch then names the harvest.
        bounds = np.cumsum([0] + r.new_unique)
        out[name] = {"instance": inst_name, "config": cfg, "unique": r.unique,
                     "attempts": r.attempts, "restarts": r.restarts, "timed_out": r.timed_out,
                     "loss_trace": r.loss_trace, "new_unique": r.new_unique, "note": r.note,
                     "words": int(r.keys.shape[1]) if r.keys.ndim == 2 else 0,
                     "keys_sha256": sha(r.keys),
                     "harvest_sha256": [sha(r.keys[bounds[i]:bounds[i + 1]])
                                        for i in range(len(r.new_unique))],
                     "first_key": [f"{int(w):016x}" for w in r.keys[0]] if r.unique else [],
                     "ref_wall_s": r.wall, "ref_threads": threads}
        print(f"{name}: unique {r.unique} attempts {r.attempts} new {r.new_unique} "
              f"({time.time() - t0:.1f}s)", flush=True)
        with open(OUT, "w") as f:
            json.dump(out, f, indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or list(BENCH_RUNS))
