"""Generates the committed instances and golden vectors from the REFERENCE.

Run in the build container (needs /root/reference, via oracle/_ref):

    make -C oracle && python tests/golden/make_fixtures.py

Outputs
* data/instances/<name>.cnf.gz / .circuit.json.gz -- the reference's own
  write_dimacs (cnf.cpp:109-127) and export_json (circuit.cpp:179-210) of each
  synthetic instance, plus a "satgrad_b200" meta
  key (generator, unsat flag).  These are what bench.py and the GPU tests
  load on the GPU box, where /root/reference does not exist.
* tests/golden/corpus.json.gz -- the acceptance corpus shapes
  (acceptance_main.cpp:47-97) as DIMACS + circuit JSON.
* tests/golden/runs.json -- satgrad::run (f32) results on fixed configs:
  stats, loss traces, per-harvest new-unique counts, and the insertion-ordered
  solution keys (full for small runs, sha256 for large ones).
* tests/golden/autodiff.json + autodiff_small.npz -- forward tape / y and
  backward dv / dp of the reference f32 path on seeded V (sha256 of the raw
  arrays; full arrays for the small instances).
"""
from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import RefInstance, RefLib  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "data", "instances")
MUX = "/root/reference/proj/tests/data/mux_chain14.cnf"

# name -> (generator, params); SURVEY.md section 8 table.
INSTANCES = {
    "mux_chain14": ("dimacs_file", MUX),
    "single_model": ("dimacs", "p cnf 2 2\n1 0\n-2 0\n"),          # test_sampler.cpp:159-170
    "unsat_unit": ("dimacs", "p cnf 1 2\n1 0\n-1 0\n"),             # test_sampler.cpp:172-180
    "free_inputs": ("dimacs", "p cnf 4 5\n3 0\n-1 -2 4 0\n-1 2 -4 0\n1 -3 4 0\n1 3 -4 0\n"),
    "c1a_planted3sat": ("planted_3sat", (1, 100, 400)),
    "c1b_random": ("random_circuit", (1, 20, 8, 10, 4)),
    "c2_iscas": ("random_circuit", (15850, 600, 40, 240, 7)),
    "c3a_or50": ("or_chain", (424242, 50, 5, 10, 4, 4)),
    "c3b_or100": ("or_chain", (99, 98, 5, 20, 4, 10)),
    "c4_blasted": ("random_circuit", (31337, 400, 400, 100, 2)),
}

# TKind enum order of tests/gen.hpp:20 and the acceptance signature ranges.
SIGS = [(0, "not", 1, 1), (1, "buf", 1, 1), (2, "and", 2, 8), (3, "or", 2, 8),
        (4, "nand", 2, 8), (5, "nor", 2, 8), (6, "xor", 2, 8), (7, "xnor", 2, 8),
        (8, "mux", 3, 3)]
SHAPES = [(4, 3, 2), (5, 3, 2), (4, 4, 2), (5, 4, 2), (4, 5, 2), (4, 3, 3), (5, 3, 3), (4, 4, 3)]

# (instance, config) golden runs; configs follow the reference tests.
RUNS = [
    ("mux_chain14", dict(batch=64, seed=7)),                                   # test_sampler :97
    ("mux_chain14", dict(batch=128, seed=9)),                                  # :116
    ("mux_chain14", dict(batch=64, seed=3, max_solutions=1000, restart=True)),  # :132
    ("mux_chain14", dict(batch=64, seed=5, max_solutions=3)),                  # :149
    ("mux_chain14", dict(batch=64, seed=21)),                                  # :193
    ("single_model", dict(batch=4, max_solutions=1, restart=True)),            # :159
    ("unsat_unit", dict(batch=1024)),                                          # :172
    ("free_inputs", dict(batch=8, iterations=3, seed=2)),                      # :205
    ("c3a_or50", dict(batch=10000, seed=1)),                                   # acceptance C7
    ("c3a_or50", dict(batch=1000, iterations=8, seed=1)),                      # C8
    ("c3a_or50", dict(batch=512, iterations=4, seed=123)),                     # C9
    ("c3a_or50", dict(batch=4096, seed=1, max_solutions=1000, restart=True)),  # bench semantics
    ("c3b_or100", dict(batch=4096, seed=1)),
    ("c1b_random", dict(batch=1024, seed=1)),
    ("c1b_random", dict(batch=1024, seed=1, max_solutions=1000, restart=True)),
    ("c1a_planted3sat", dict(batch=1024, seed=1)),
    ("c2_iscas", dict(batch=512, iterations=2, seed=1)),
    ("c4_blasted", dict(batch=128, iterations=1, seed=1)),
]

AUTODIFF = [("mux_chain14", 64, 11), ("c3a_or50", 256, 11), ("c1b_random", 256, 5),
            ("c1a_planted3sat", 64, 3), ("c2_iscas", 64, 1), ("c4_blasted", 16, 1)]
SMALL_AD = {"mux_chain14", "c3a_or50", "c1b_random"}


def make(gen, param) -> RefInstance:
    if gen == "dimacs_file":
        return RefInstance.from_dimacs(open(param).read())
    if gen == "dimacs":
        return RefInstance.from_dimacs(param)
    return getattr(RefInstance, gen)(*param)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def meta_json(inst: RefInstance, meta: dict) -> str:
    j = json.loads(inst.circuit_json())
    j["satgrad_b200"] = dict(meta, unsat=inst.unsat, unsat_note=inst.unsat_note,
                             constrained_pi=[int(x) for x in inst.cpi],
                             unconstrained_pi=[int(x) for x in inst.ucpi])
    return json.dumps(j, separators=(",", ":")) + "\n"


def write_gz(path: str, text: str) -> None:
    with gzip.GzipFile(path, "wb", mtime=0) as f:  # reproducible bytes
        f.write(text.encode())


def main() -> None:
    os.makedirs(DATA, exist_ok=True)
    insts = {}
    for name, (gen, param) in INSTANCES.items():
        inst = make(gen, param)
        insts[name] = inst
        meta = {"generator": gen, "params": param if gen != "dimacs_file" else "mux_chain14.cnf"}
        write_gz(os.path.join(DATA, name + ".cnf.gz"), inst.dimacs())
        write_gz(os.path.join(DATA, name + ".circuit.json.gz"), meta_json(inst, meta))
        print(f"{name}: vars {inst.num_vars} clauses {inst.n_clauses} nodes {inst.n_nodes} "
              f"cpi {inst.n_cpi} ucpi {inst.n_ucpi} outputs {inst.n_out} unsat {inst.unsat}")

    corpus = []
    for tk, nm, lo, hi in SIGS:
        for n in range(lo, hi + 1):
            inst = RefInstance.gate_signature(tk, n)
            corpus.append({"name": f"{nm}{n}", "cnf": inst.dimacs(),
                           "circuit": meta_json(inst, {"generator": "gate_signature",
                                                       "params": [tk, n]})})
    for i in range(110):
        sh = SHAPES[i % len(SHAPES)]
        inst = RefInstance.random_circuit(1000 + i, sh[0], sh[1], sh[2], 2)
        corpus.append({"name": f"random{i}", "cnf": inst.dimacs(),
                       "circuit": meta_json(inst, {"generator": "random_circuit",
                                                   "params": [1000 + i, *sh, 2]})})
    corpus_runs = []
    for entry in corpus:  # acceptance criterion 2 config
        inst = RefInstance.from_dimacs(entry["cnf"])
        r = inst.run(batch=128, iterations=3, seed=1)
        entry["run"] = {"unique": r.unique, "attempts": r.attempts, "new_unique": r.new_unique,
                        "loss_trace": r.loss_trace,
                        "keys": [[f"{int(w):016x}" for w in k] for k in r.keys]}
        corpus_runs.append(r.unique)
    write_gz(os.path.join(GOLDEN, "corpus.json.gz"), json.dumps(corpus, separators=(",", ":")))
    print(f"corpus: {len(corpus)} instances, {sum(corpus_runs)} solutions")

    runs = []
    for name, cfg in RUNS:
        r = insts[name].run(use_f32=True, **cfg)
        rec = {"instance": name, "config": cfg, "unique": r.unique, "attempts": r.attempts,
               "restarts": r.restarts, "timed_out": r.timed_out, "loss_trace": r.loss_trace,
               "new_unique": r.new_unique, "note": r.note, "keys_sha256": sha(r.keys),
               "wall_s": r.wall}
        if r.keys.size <= 20000:
            rec["keys"] = [[f"{int(w):016x}" for w in k] for k in r.keys]
        runs.append(rec)
        print(f"run {name} {cfg}: unique {r.unique} attempts {r.attempts} ({r.wall:.2f}s)")
    with open(os.path.join(GOLDEN, "runs.json"), "w") as f:
        json.dump(runs, f, indent=1)

    lib = RefLib()
    ad, small = [], {}
    for name, batch, seed in AUTODIFF:
        inst = insts[name]
        v = lib.init_soft_inputs(batch, inst.n_cpi, seed).astype(np.float32)
        p = lib.embed_f32(v).reshape(v.shape)
        tape, y = inst.forward(inst.cpi, p)
        dv, dp = inst.backward(inst.cpi, tape, inst.out_tgt, v)
        per_row, total = lib.loss_f32(y, inst.out_tgt)
        ad.append({"instance": name, "batch": batch, "seed": seed, "v": sha(v), "p": sha(p),
                   "tape": sha(tape), "y": sha(y), "dv": sha(dv), "dp": sha(dp),
                   "row_loss": sha(per_row), "loss_total": total})
        if name in SMALL_AD:
            for k, arr in (("v", v), ("p", p), ("tape", tape), ("y", y), ("dv", dv), ("dp", dp),
                           ("row_loss", per_row)):
                small[f"{name}.{k}"] = arr
    with open(os.path.join(GOLDEN, "autodiff.json"), "w") as f:
        json.dump(ad, f, indent=1)
    np.savez_compressed(os.path.join(GOLDEN, "autodiff_small.npz"), **small)

    # rng.hpp known answers
    rng = {"hash5": [], "hash6": []}
    for t in [(1, 0x696e6974, 0, 0, 0), (7, 0x696e6974, 3, 12345, 17), (2**63 + 5, 1, 2, 3, 4)]:
        rng["hash5"].append([list(map(str, t)), str(lib.hash5(*t))])
    for t in [(1, 0x66726565, 0, 1, 2, 3), (9, 0x66726565, 4, 5, 65535, 84)]:
        rng["hash6"].append([list(map(str, t)), str(lib.hash6(*t))])
    rng["init_1x4_seed42"] = lib.init_soft_inputs(2, 4, 42, 1).ravel().tolist()
    with open(os.path.join(GOLDEN, "rng.json"), "w") as f:
        json.dump(rng, f, indent=1)


if __name__ == "__main__":
    main()
