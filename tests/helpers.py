"""Shared test helpers: golden fixtures and the oracle front ends."""
from __future__ import annotations

import gzip
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def golden_runs():
    with open(os.path.join(GOLDEN, "runs.json")) as f:
        return json.load(f)


def golden_autodiff():
    with open(os.path.join(GOLDEN, "autodiff.json")) as f:
        return json.load(f)


def golden_small():
    return np.load(os.path.join(GOLDEN, "autodiff_small.npz"))


def golden_corpus():
    with gzip.open(os.path.join(GOLDEN, "corpus.json.gz"), "rt") as f:
        return json.load(f)


def keys_from_hex(rows) -> np.ndarray:
    if not rows:
        return np.zeros((0, 0), np.uint64)
    return np.array([[int(w, 16) for w in r] for r in rows], np.uint64)


def sha(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def cfg_kwargs(cfg: dict) -> dict:
    """runs.json config -> SamplerConfig kwargs."""
    from paper_2502_08673_b200 import RestartPolicy
    out = dict(cfg)
    if out.pop("restart", False):
        out["restart"] = RestartPolicy.REINIT_ON_EXHAUST
    return out


def instance_from_corpus(entry):
    from paper_2502_08673_b200 import Instance, classify_paths, import_json, parse_dimacs
    cnf = parse_dimacs(entry["cnf"])
    c = import_json(entry["circuit"])
    meta = json.loads(entry["circuit"]).get("satgrad_b200", {})
    return Instance(entry["name"], cnf, c, classify_paths(c), bool(meta.get("unsat", False)))


def init_v(batch, cols, seed, restart=0) -> np.ndarray:
    """init_soft_inputs through the C port oracle, cast to f32."""
    from oracle.oracle import PortLib
    return PortLib().init_soft_inputs(batch, cols, seed, restart).astype(np.float32)
