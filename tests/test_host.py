"""CPU tests of the host side: the C-ABI library loads and exports its header,
the host levelizer / layout compiler, DIMACS and circuit-JSON I/O (mirroring
the reference's test_cnf.cpp / test_circuit.cpp expectations), path
classification against the reference's own classify_paths, and the host
re-verifier.  No device calls."""
import ctypes as C
import gzip
import json
import os
import re

import numpy as np
import pytest

from helpers import ROOT, golden_runs, keys_from_hex
from paper_2502_08673_b200 import (ParseError, SchemaError, classify_paths, eval_cnf, export_json,
                                   import_json, layout_stats, load_instance, parse_dimacs,
                                   verify_keys, write_dimacs)
from paper_2502_08673_b200 import _lib
from paper_2502_08673_b200.cnf import format_solution_line, key_to_assignment

MUX = os.path.join(ROOT, "data", "instances", "mux_chain14.cnf.gz")


def mux_text():
    with gzip.open(MUX, "rt") as f:
        return f.read()


def test_library_exports_every_header_symbol():
    L = _lib.load()
    header = open(os.path.join(ROOT, "include", "satgrad_b200.h")).read()
    declared = set(re.findall(r"\b(sgx_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_lib.EXPORTS)
    for name in declared:
        assert getattr(L, name) is not None
    assert L.sgx_version().startswith(b"satgrad_b200")


def test_library_is_sm100a():
    data = open(_lib.library_path(), "rb").read()
    assert b"sm_100a" in data


def test_parse_mux_fixture():  # test_cnf.cpp "dimacs parse of the mux chain fixture"
    cnf = parse_dimacs(mux_text())
    assert cnf.num_vars == 14 and cnf.n_clauses == 21 and len(cnf.comments) == 10
    cl = list(cnf.clauses())
    assert cl[0] == [-1, -2] and cl[-1] == [10]


def test_write_parse_round_trip():
    cnf = parse_dimacs(mux_text())
    again = parse_dimacs(write_dimacs(cnf))
    assert again.num_vars == cnf.num_vars
    assert list(again.clauses()) == list(cnf.clauses())
    assert again.comments == cnf.comments


def test_parse_edge_cases():
    cnf = parse_dimacs("p cnf 2 1\n1 -2 0")  # final clause at EOF
    assert list(cnf.clauses()) == [[1, -2]]
    assert list(parse_dimacs("p cnf 2 1\n1 1 -2 1 0\n").clauses()) == [[1, -2]]
    warnings = []
    cnf = parse_dimacs("p cnf 2 5\n1 0\n-2 0\n", warnings)
    assert cnf.n_clauses == 2 and "declares 5" in warnings[0]
    for bad in ["p cnf nope 1\n", "1 2 0\np cnf 2 1\n", "p cnf 2 1\n1 -3 0\n", "p cnf 2 1\n1 2\n",
                "p cnf 2 1\n0\n", "p cnf 2 1\np cnf 2 1\n", "", "p cnf 2 1\n1 x 0\n"]:
        with pytest.raises(ParseError):
            parse_dimacs(bad)


def test_eval_cnf():
    cnf = parse_dimacs("p cnf 3 2\n1 -2 0\n2 3 0\n")
    a = np.array([0xFF, 1, 1, 0], np.uint8)
    assert eval_cnf(cnf, a)
    a[1] = 0
    assert not eval_cnf(cnf, a)
    a[1] = 0xFF
    with pytest.raises(ValueError):
        eval_cnf(cnf, a)


def test_key_helpers():  # test_sampler.cpp key packing / line format
    key = np.array([(1 << 0) | (1 << 63), 1 << 5], np.uint64)
    a = key_to_assignment(key, 70)
    assert a[1] == 1 and a[64] == 1 and a[70] == 1 and a[2] == 0
    assert format_solution_line(np.array([0b101], np.uint64), 3) == "1 -2 3 0"


def test_verify_keys_matches_golden_solutions():
    inst = load_instance("c3a_or50")
    rec = [r for r in golden_runs() if r["instance"] == "c3a_or50" and "keys" in r][0]
    keys = keys_from_hex(rec["keys"])
    assert verify_keys(inst.cnf, keys).all()
    bad = keys.copy()
    bad[:, 0] ^= np.uint64(0xFFFF)  # flip 16 inputs: most rows now violate a clause
    assert not verify_keys(inst.cnf, bad).all()


@pytest.mark.parametrize("name", ["mux_chain14", "c1a_planted3sat", "c1b_random", "c2_iscas",
                                  "c3a_or50", "c3b_or100", "c4_blasted", "free_inputs",
                                  "single_model"])
def test_classify_paths_matches_reference(name):
    inst = load_instance(name)
    with gzip.open(os.path.join(ROOT, "data", "instances", name + ".circuit.json.gz"), "rt") as f:
        meta = json.load(f)["satgrad_b200"]
    pc = classify_paths(inst.circuit)
    assert list(pc.constrained_pi) == meta["constrained_pi"]
    assert list(pc.unconstrained_pi) == meta["unconstrained_pi"]


def test_circuit_json_round_trip():
    inst = load_instance("c1b_random")
    again = import_json(export_json(inst.circuit))
    for f in ("kind", "a", "b", "var", "inputs", "out_var", "out_tgt"):
        assert np.array_equal(getattr(again, f), getattr(inst.circuit, f))


def test_circuit_json_schema_errors():  # circuit.cpp import_json checks
    good = json.loads(export_json(load_instance("mux_chain14").circuit))
    for mutate in (lambda j: j.update(aux_base=j["num_vars"] + 1),
                   lambda j: j["gates"][3].update(id=7),
                   lambda j: j["gates"][5].update(kind="NAND"),
                   lambda j: j["gates"][6].update(args=[6]),
                   lambda j: j["outputs"].append(dict(j["outputs"][0])),
                   lambda j: j["inputs"].append(999)):
        j = json.loads(json.dumps(good))
        mutate(j)
        with pytest.raises(SchemaError):
            import_json(json.dumps(j))
    with pytest.raises(SchemaError):
        import_json("{not json")


# SURVEY.md section 8 structure figures for the configs (cone nodes / edges / levels).
@pytest.mark.parametrize("name,cone,edges,levels", [("c2_iscas", 13453, 20152, 92),
                                                    ("c4_blasted", 66317, 102713, 877),
                                                    ("c3a_or50", 218, 294, 18),
                                                    ("c3b_or100", 490, 636, 19)])
def test_levelizer_matches_survey_structure(name, cone, edges, levels):
    inst = load_instance(name)
    st = layout_stats(inst.cnf, inst.circuit, inst.paths)
    assert st["cone_nodes"] == cone
    assert st["cone_edges"] == edges
    assert st["bit_levels"] == levels
    # NOT/BUF folding shrinks the tape and the level count of the soft program.
    assert st["fwd_ops"] < cone and st["soft_levels"] < levels
    assert st["key_words"] == (inst.num_vars + 63) // 64


def test_layout_rejects_what_the_reference_rejects():
    inst = load_instance("c3a_or50")
    c = inst.circuit
    # an operand that is not an earlier node (circuit.hpp:28)
    bad = type(c)(c.num_vars, c.kind.copy(), c.a.copy(), c.b.copy(), c.var.copy(), c.inputs,
                  c.out_var, c.out_tgt)
    j = int(np.nonzero(bad.kind >= 5)[0][0])
    bad.a[j] = j
    with pytest.raises(ValueError, match="earlier"):
        layout_stats(inst.cnf, bad, inst.paths)
    # a V column that is not a circuit input (autodiff.cpp:44-46)
    from paper_2502_08673_b200 import PathClassification
    gate_var = int(c.var[np.nonzero((c.kind >= 3) & (c.var > 0))[0][0]])
    pc = PathClassification(np.append(inst.paths.constrained_pi, gate_var).astype(np.int32),
                            inst.paths.unconstrained_pi)
    with pytest.raises(ValueError, match="not a circuit input"):
        layout_stats(inst.cnf, c, pc)


def test_unsat_instance_is_flagged():
    inst = load_instance("unsat_unit")
    assert inst.unsat and inst.unsat_note


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2502_08673_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cpp", ".cu", ".cuh", ".hpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "from oracle" not in src, f
                assert "libsgx_oracle" not in src and "libsatgrad_ref" not in src, f
