"""Native circuit extraction (csrc/sgx_extract.cpp) against
the reference's extract + build (src/extract.cpp:43-172, src/circuit.cpp:
60-122).

1. Golden: every committed instance (data/instances, the 60-instance C5 suite,
   the 155-instance acceptance corpus) carries the circuit the reference built
   for its CNF; the native extractor must rebuild it node for node, with the
   same PI / PO orders and the same unsat verdict and note.
2. Live: random CNFs (unit clauses, tautologies, repeated literals, gate
   encodings mixed with noise, contradictions) through the reference library
   (oracle/_ref) and the native path; circuits and ExtractionResult lists
   (iv, aux) must be identical.

Host-only: no GPU needed (the library loads without one).
"""
import glob
import os

import numpy as np
import pytest

from helpers import golden_corpus
from paper_2502_08673_b200 import (CnfFormula, extract_circuit, instance_from_cnf, load_instance,
                                   parse_dimacs, write_dimacs)
from paper_2502_08673_b200.circuit import DATA_DIR

FIELDS = ("kind", "a", "b", "var", "inputs", "out_var", "out_tgt")


def _names():
    out = [os.path.basename(p)[:-7] for p in sorted(glob.glob(DATA_DIR + "/*.cnf.gz"))]
    out += ["c5/" + os.path.basename(p)[:-7] for p in sorted(glob.glob(DATA_DIR + "/c5/*.cnf.gz"))]
    return out


def _same(c, ref):
    for f in FIELDS:
        x, y = np.asarray(getattr(c, f)), np.asarray(getattr(ref, f))
        assert x.shape == y.shape and np.array_equal(x, y), f


@pytest.mark.parametrize("name", _names())
def test_extract_matches_golden_instances(name):
    inst = load_instance(name)
    r = extract_circuit(inst.cnf)
    _same(r.circuit, inst.circuit)
    assert r.unsat == inst.unsat
    if inst.unsat:
        assert r.unsat_note == inst.unsat_note


def test_extract_matches_golden_corpus():
    from helpers import instance_from_corpus
    corpus = golden_corpus()
    entries = corpus["instances"] if isinstance(corpus, dict) and "instances" in corpus else corpus
    n = 0
    for e in entries:
        inst = instance_from_corpus(e)
        r = extract_circuit(inst.cnf)
        _same(r.circuit, inst.circuit)
        assert r.unsat == inst.unsat, e["name"]
        n += 1
    assert n >= 100


def _random_cnf(rng, nv, nc):
    clauses = []
    for _ in range(nc):
        r = rng.random()
        if r < 0.08:  # unit
            clauses.append([int(rng.integers(1, nv + 1)) * int(rng.choice([-1, 1]))])
        elif r < 0.45:  # a gate encoding: z = AND/OR/XOR of two vars
            z, x, y = (int(v) for v in rng.choice(np.arange(1, nv + 1), 3, replace=False))
            g = rng.integers(0, 3)
            if g == 0:
                clauses += [[-z, x], [-z, y], [z, -x, -y]]
            elif g == 1:
                clauses += [[z, -x], [z, -y], [-z, x, y]]
            else:
                clauses += [[-z, x, y], [-z, -x, -y], [z, -x, y], [z, x, -y]]
        else:
            k = int(rng.integers(1, 6))
            vs = rng.integers(1, nv + 1, k)  # repeats and tautologies allowed
            clauses.append([int(v) * int(rng.choice([-1, 1])) for v in vs])
    return CnfFormula.from_clauses(nv, clauses)


@pytest.mark.parametrize("seed", range(40))
def test_extract_matches_reference_random(seed):
    from oracle.oracle import RefInstance, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(seed)
    nv = int(rng.integers(3, 40))
    cnf = _random_cnf(rng, nv, int(rng.integers(1, 4 * nv)))
    text = write_dimacs(cnf)
    ref = RefInstance.from_dimacs(text)
    r = extract_circuit(parse_dimacs(text))
    _same(r.circuit, ref)
    assert r.unsat == ref.unsat
    assert r.unsat_note == ref.unsat_note
    sizes, iv, aux = ref.extraction_lists()
    assert [len(r.pi), len(r.po_var), len(r.iv), len(r.aux), r.n_defs] == sizes
    assert np.array_equal(r.iv, iv) and np.array_equal(r.aux, aux)


def test_extract_matches_reference_generated():
    """Generator-built CNFs (random circuits, or-chains, every gate signature)."""
    from oracle.oracle import RefInstance, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    refs = [RefInstance.random_circuit(s, 12, 6, 8, 3) for s in range(6)]
    refs += [RefInstance.or_chain(s, 20, 4, 6, 3, 2) for s in range(4)]
    refs += [RefInstance.gate_signature(t, a) for t in range(6) for a in (2, 3, 4)]
    for ref in refs:
        r = extract_circuit(parse_dimacs(ref.dimacs()))
        _same(r.circuit, ref)
        assert r.unsat == ref.unsat


def test_instance_from_cnf_equals_cached_instance():
    inst = load_instance("c3a_or50")
    path = os.path.join(DATA_DIR, "c3a_or50.cnf.gz")
    got = instance_from_cnf(path)
    _same(got.circuit, inst.circuit)
    assert np.array_equal(got.paths.constrained_pi, inst.paths.constrained_pi)
    assert np.array_equal(got.paths.unconstrained_pi, inst.paths.unconstrained_pi)


def test_extract_rejects_bad_input():
    bad = CnfFormula(2, np.array([0, 2], np.int64), np.array([1, 3], np.int32))
    with pytest.raises(ValueError):
        extract_circuit(bad)
    with pytest.raises(ValueError):
        extract_circuit(CnfFormula.from_clauses(3, [[1, 2]]), minimize_cap=17)


def test_extract_empty_and_trivial():
    r = extract_circuit(CnfFormula.from_clauses(3, []))
    assert list(r.pi) == [1, 2, 3] and len(r.po_var) == 0 and r.circuit.n_nodes == 3
    r = extract_circuit(CnfFormula.from_clauses(2, [[1], [-1]]))
    assert r.unsat and "forced" in r.unsat_note


@pytest.mark.parametrize("name", ["c1b_random", "c2_iscas", "c4_blasted", "mux_chain14", "unsat_unit",
                                  "free_inputs", "single_model"])
def test_reference_adapter_extract_drop_in(tmp_path, name):
    """include/satgrad_b200_adapter.hpp's satgrad_b200::extract inside the
    UNMODIFIED reference pipeline (oracle/adapter_check.cpp --extract-only):
    Circuit, ExtractionResult lists and PathClassification equal the
    reference's extract + build + classify_paths."""
    import gzip
    import subprocess
    from helpers import ROOT
    exe = os.path.join(ROOT, "oracle", "_ref", "adapter_check")
    if not os.path.exists(exe):
        pytest.skip("adapter check not built (make -C oracle adapter)")
    cnf = tmp_path / f"{name}.cnf"
    cnf.write_bytes(gzip.open(os.path.join(DATA_DIR, f"{name}.cnf.gz")).read())
    r = subprocess.run([exe, str(cnf), "--extract-only"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0 and "extract ok" in r.stdout, r.stdout + r.stderr


@pytest.mark.parametrize("ccap,mcap", [(0, 12), (2, 0), (4, 2), (8, 6), (16, 16), (40, 12)])
def test_extract_caps_match_reference(ccap, mcap):
    """Non-default ExtractorConfig (extract.hpp:14-17): the complement-check cap
    (clamped to the 16-variable truth-table limit, boolexpr.cpp:271-283) and
    the two-level minimisation cap change which definitions are found and how
    they are simplified; the circuit must still match the reference's."""
    from oracle.oracle import RefInstance, ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    cnfs = [load_instance(n).cnf for n in ("c1b_random", "mux_chain14", "c3a_or50")]
    rng = np.random.default_rng(ccap * 31 + mcap)
    cnfs += [_random_cnf(rng, int(rng.integers(5, 30)), int(rng.integers(5, 80))) for _ in range(8)]
    for cnf in cnfs:
        text = write_dimacs(cnf)
        ref = RefInstance.from_dimacs_cfg(text, ccap, mcap)
        r = extract_circuit(parse_dimacs(text), complement_cap=ccap, minimize_cap=mcap)
        _same(r.circuit, ref)
        assert r.unsat == ref.unsat and r.unsat_note == ref.unsat_note
