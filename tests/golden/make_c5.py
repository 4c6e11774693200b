"""Generates the C5 suite (BASELINE.json configs[4]):
60 synthetic instances of the paper's benchmark families, built by the
REFERENCE's own generators (tests/gen.cpp via oracle/_ref), plus the
reference's satgrad::run (f32) on each at a small batch as golden vectors.

Run in the build container (needs /root/reference):

    make -C oracle ref && python tests/golden/make_c5.py

Families (seeds 1..60, one per instance):
*  1-16 or-chain shaped: or_chain(seed, inputs in {50,60,70,100}, levels 5,
         gpl in {10,20}, arity 4, outs in {4,5,7,10})
* 17-32 q-shaped: random_circuit(seed, 300, 3, 50, 1) (~450 vars, 1 output)
* 33-44 s15850-shaped: random_circuit(seed, 600, 40, 230, outs in {3,7,15})
* 45-54 Prod-shaped: random_circuit(seed, 1000-1540, 20-26, 700-1060, 5)
         (15k-29k vars; the reference generator gives ~3.1 clauses per var,
         so these carry 46k-91k clauses)
* 55-60 blasted-shaped (deep): random_circuit(seed, 300, levels in
         {200,300,450,600,750,900}, gpl 80..30, 2)

Outputs
* data/instances/c5/<name>.cnf.gz / .circuit.json.gz (reference write_dimacs /
  export_json, as for the other instances) and data/instances/c5/manifest.json
* tests/golden/c5_runs.json: per instance satgrad::run(batch 256, 5
  iterations, seed 1, f32): unique count, attempts, per-harvest new-unique
  trace, loss trace, sha256 of the insertion-ordered keys.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

from make_fixtures import GOLDEN, meta_json, sha, write_gz  # noqa: E402
from oracle.oracle import RefInstance  # noqa: E402

C5_DIR = os.path.join(ROOT, "data", "instances", "c5")
RUN_CFG = dict(batch=256, iterations=5, seed=1)


def suite():
    out = []
    for i in range(16):
        seed = 1 + i
        p = (seed, [50, 60, 70, 100][i % 4], 5, [10, 20][(i // 4) % 2], 4, [4, 5, 7, 10][(i // 2) % 4])
        out.append((f"or{p[1]}_{seed:02d}", "or_chain", p))
    for i in range(16):
        seed = 17 + i
        out.append((f"q_{seed:02d}", "random_circuit", (seed, 300, 3, 50, 1)))
    for i in range(12):
        seed = 33 + i
        out.append((f"s15850_{seed:02d}", "random_circuit", (seed, 600, 40, 230, [3, 7, 15][i % 3])))
    for i in range(10):
        seed = 45 + i
        out.append((f"prod_{seed:02d}", "random_circuit",
                    (seed, 1000 + 60 * i, 20 + (6 * i) // 9, 700 + 40 * i, 5)))
    for i, (lv, gpl) in enumerate([(200, 80), (300, 60), (450, 50), (600, 40), (750, 36), (900, 30)]):
        seed = 55 + i
        out.append((f"blasted{lv}_{seed:02d}", "random_circuit", (seed, 300, lv, gpl, 2)))
    return out


def main() -> None:
    os.makedirs(C5_DIR, exist_ok=True)
    manifest, runs = [], []
    for name, gen, param in suite():
        inst = getattr(RefInstance, gen)(*param)
        meta = {"generator": gen, "params": list(param), "suite": "c5"}
        write_gz(os.path.join(C5_DIR, name + ".cnf.gz"), inst.dimacs())
        write_gz(os.path.join(C5_DIR, name + ".circuit.json.gz"), meta_json(inst, meta))
        r = inst.run(use_f32=True, **RUN_CFG)
        manifest.append({"name": "c5/" + name, "generator": gen, "params": list(param),
                         "vars": inst.num_vars, "clauses": inst.n_clauses, "nodes": inst.n_nodes,
                         "cpi": inst.n_cpi, "outputs": inst.n_out, "unsat": inst.unsat})
        runs.append({"instance": "c5/" + name, "config": RUN_CFG, "unique": r.unique,
                     "attempts": r.attempts, "restarts": r.restarts, "loss_trace": r.loss_trace,
                     "new_unique": r.new_unique, "keys_sha256": sha(r.keys), "wall_s": r.wall})
        print(f"{name}: vars {inst.num_vars} clauses {inst.n_clauses} nodes {inst.n_nodes} "
              f"unique {r.unique} ({r.wall:.2f}s)", flush=True)
    with open(os.path.join(C5_DIR, "manifest.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    with open(os.path.join(GOLDEN, "c5_runs.json"), "w") as f:
        json.dump(runs, f, indent=1)


if __name__ == "__main__":
    main()
