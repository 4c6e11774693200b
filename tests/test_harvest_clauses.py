"""Harvest clause pruning (sgx_layout.cpp harvest_clauses), host only.

The harvest skips CNF clauses that every row passing eval_discrete + the
output check satisfies (cnf.cpp:129-147 would find them true).  The layout
compiler proves that per clause from a small truth table; here an independent
check holds it to the circuit's own semantics: each skipped clause either has
a literal an output target forces true, or is satisfied on every one of
16,384 random input assignments with all gates evaluated as in
eval_discrete (circuit.cpp:124-152).  The GPU goldens (bench-size and corpus
runs) show the verdicts are unchanged end to end.
"""
import numpy as np
import pytest

from helpers import golden_corpus, instance_from_corpus
from paper_2502_08673_b200 import load_instance
from paper_2502_08673_b200.circuit import Circuit, Instance, PathClassification
from paper_2502_08673_b200.cnf import CnfFormula
from paper_2502_08673_b200.sampler import harvest_clause_mask

W = 256  # 64-row words: 16,384 random rows


def simulate(circuit, seed=0):
    """Bit-parallel eval_discrete on random inputs: value words per node."""
    rng = np.random.default_rng(seed)
    kind, a, b = circuit.kind, circuit.a, circuit.b
    val = np.zeros((circuit.n_nodes, W), np.uint64)
    for i in range(circuit.n_nodes):
        k = int(kind[i])
        if k == 0:
            val[i] = rng.integers(0, 1 << 64, W, dtype=np.uint64, endpoint=False)
        elif k == 1:
            val[i] = 0
        elif k == 2:
            val[i] = ~np.uint64(0)
        elif k == 3:
            val[i] = val[a[i]]
        elif k == 4:
            val[i] = ~val[a[i]]
        elif k == 5:
            val[i] = val[a[i]] & val[b[i]]
        elif k == 6:
            val[i] = val[a[i]] | val[b[i]]
        elif k == 7:
            val[i] = val[a[i]] ^ val[b[i]]
        else:
            val[i] = ~(val[a[i]] ^ val[b[i]])
    return val


def check_sound(inst):
    mask = harvest_clause_mask(inst.cnf, inst.circuit, inst.paths, inst.unsat)
    cnf, c = inst.cnf, inst.circuit
    assert mask.shape == (len(cnf.clause_ptr) - 1,)
    if not mask.any():
        return mask
    val = simulate(c)
    node_of_var = {int(v): i for i, v in enumerate(c.var) if v > 0}
    forced = {int(v): int(t) for v, t in zip(c.out_var, c.out_tgt)}
    ones = ~np.uint64(0)
    for ci in np.flatnonzero(mask):
        lits = cnf.clause_lit[cnf.clause_ptr[ci]:cnf.clause_ptr[ci + 1]]
        if any(abs(int(l)) in forced and forced[abs(int(l))] == (1 if l > 0 else 0) for l in lits):
            continue
        acc = np.zeros(W, np.uint64)
        for l in lits:
            x = val[node_of_var[abs(int(l))]]
            acc |= x if l > 0 else ~x
        assert (acc == ones).all(), f"clause {ci} {list(lits)} skipped but violated"
    return mask


@pytest.mark.parametrize("name", ["c1b_random", "c2_iscas", "c3a_or50", "c3b_or100"])
def test_pruned_clauses_hold_on_bench_instances(name):
    mask = check_sound(load_instance(name))
    assert mask.mean() > 0.9  # gate-structured CNFs: nearly every clause is a definition


def test_pruned_clauses_hold_on_corpus():
    n_kept = n_skipped = 0
    for entry in golden_corpus():
        inst = instance_from_corpus(entry)
        mask = check_sound(inst)
        n_skipped += int(mask.sum())
        n_kept += int((mask == 0).sum())
    assert n_skipped > 0 and n_kept > 0  # the corpus exercises both sides


def test_residual_clause_is_kept():
    """x3 = AND(x1, x2), an output with target 1, with its three definition
    clauses, plus a residual (x1 | x2) that no gate defines: only the
    residual is checked."""
    cnf = CnfFormula(num_vars=3, clause_ptr=np.array([0, 2, 4, 7, 9], np.int64),
                     clause_lit=np.array([-3, 1, -3, 2, 3, -1, -2, 1, 2], np.int32))
    circ = Circuit(num_vars=3, kind=[0, 0, 5], a=[-1, -1, 0], b=[-1, -1, 1], var=[1, 2, 3],
                   inputs=[1, 2], out_var=[3], out_tgt=[1])
    paths = PathClassification(constrained_pi=np.array([1, 2], np.int32),
                               unconstrained_pi=np.array([], np.int32))
    inst = Instance("and_plus_residual", cnf, circ, paths)
    mask = check_sound(inst)
    assert mask.tolist() == [1, 1, 1, 0]


def test_all_clauses_env_disables_pruning(monkeypatch):
    inst = load_instance("c3a_or50")
    monkeypatch.setenv("SGX_ALL_CLAUSES", "1")
    assert not harvest_clause_mask(inst.cnf, inst.circuit, inst.paths).any()
