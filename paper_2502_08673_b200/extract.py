"""CNF -> circuit, natively: the reference's ``extract`` + ``build``.

``extract_circuit`` mirrors ``satgrad::extract`` (src/extract.cpp:43-172,
include/satgrad/extract.hpp:14-53) followed by ``satgrad::build``
(src/circuit.cpp:60-122): the same ExtractionResult lists (pi, po, iv, aux,
unsat note) and the same gate-level Circuit, node for node, as the reference
produces for the CNF.  The work runs in ``libsatgrad_b200.so``
(``csrc/sgx_extract.cpp``); there is no Python fallback.

``instance_from_cnf`` is what a reference user without a ``.circuit.json``
cache calls: DIMACS text or path -> Instance ready for ``run``.
"""
from __future__ import annotations

import ctypes as C
import gzip
from dataclasses import dataclass

import numpy as np

from . import _lib
from .circuit import Circuit, Instance, classify_paths
from .cnf import CnfFormula, parse_dimacs


@dataclass
class ExtractionResult:
    """extract.hpp:31-41 (expressions are built into ``circuit``)."""
    num_vars: int
    pi: np.ndarray
    iv: np.ndarray
    po_var: np.ndarray
    po_target: np.ndarray
    aux: np.ndarray
    n_defs: int
    unsat: bool
    unsat_note: str
    circuit: Circuit


def extract_circuit(cnf: CnfFormula, complement_cap: int = 16, minimize_cap: int = 12) -> ExtractionResult:
    """``build(extract(cnf, {complement_cap, minimize_cap}))``."""
    L = _lib.load()
    ptr = np.ascontiguousarray(cnf.clause_ptr, np.int64)
    if len(ptr) and ptr[-1] > np.iinfo(np.int32).max:
        raise ValueError("CNF too large for 32-bit clause offsets")
    ptr32 = ptr.astype(np.int32)
    lit = np.ascontiguousarray(cnf.clause_lit, np.int32)
    h = C.c_void_p()
    _lib.check(L.sgx_extract(int(cnf.num_vars), _lib.ptr(ptr32, C.c_int32), _lib.ptr(lit, C.c_int32),
                             int(cnf.n_clauses), int(complement_cap), int(minimize_cap), C.byref(h)))
    try:
        sz = np.zeros(7, np.int64)
        _lib.check(L.sgx_extraction_sizes(h, _lib.ptr(sz, C.c_int64)))
        n, npi, npo, niv, naux, ndef, unsat = (int(x) for x in sz)
        kind, a, b, var = (np.zeros(n, np.int32) for _ in range(4))
        pi, iv, aux = np.zeros(npi, np.int32), np.zeros(niv, np.int32), np.zeros(naux, np.int32)
        ov, ot = np.zeros(npo, np.int32), np.zeros(npo, np.uint8)
        i32 = C.c_int32
        _lib.check(L.sgx_extraction_export(h, _lib.ptr(kind, i32), _lib.ptr(a, i32), _lib.ptr(b, i32),
                                           _lib.ptr(var, i32), _lib.ptr(pi, i32), _lib.ptr(ov, i32),
                                           _lib.ptr(ot, C.c_uint8), _lib.ptr(iv, i32), _lib.ptr(aux, i32)))
        note = L.sgx_extraction_note(h).decode()
    finally:
        L.sgx_extraction_free(h)
    circuit = Circuit(int(cnf.num_vars), kind, a, b, var, pi, ov, ot)
    return ExtractionResult(int(cnf.num_vars), pi, iv, ov, ot, aux, ndef, bool(unsat), note, circuit)


def instance_from_cnf(cnf_or_path, name: str | None = None, complement_cap: int = 16,
                      minimize_cap: int = 12) -> Instance:
    """DIMACS text / path / CnfFormula -> Instance (satgrad_main's sample path
    without a circuit cache: parse, extract, build, classify_paths)."""
    if isinstance(cnf_or_path, CnfFormula):
        cnf = cnf_or_path
    else:
        text = cnf_or_path
        if "\n" not in text and (text.endswith(".cnf") or text.endswith(".gz")):
            name = name or text
            opener = gzip.open if text.endswith(".gz") else open
            with opener(text, "rt") as f:
                text = f.read()
        cnf = parse_dimacs(text)
    res = extract_circuit(cnf, complement_cap, minimize_cap)
    return Instance(name or "cnf", cnf, res.circuit, classify_paths(res.circuit), res.unsat, res.unsat_note)
