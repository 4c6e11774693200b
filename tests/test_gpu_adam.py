"""The opt-in Adam logit update (SGX_OPT_ADAM).

Adam has no reference counterpart (SPEC.md:418 lists adaptive optimizers as
a non-goal), so its parity is UNPINNED: it is checked against a float64
numpy restatement of the textbook update, driven by the reference's own dV
(the port oracle's backward, bit-exact with the device's), with a stated
tolerance: |V_dev - V_ref| <= 2e-5 * max(1, |V_ref|) per logit per step (f32
arithmetic against f64; the update itself is at most lr in size).  The
default GD path is untouched (every other GPU test runs it).
"""
import numpy as np
import pytest

from oracle.oracle import PortLib
from paper_2502_08673_b200 import (DeviceCircuit, Optimizer, Sampler, SamplerConfig, load_instance,
                                   verify_keys)

pytestmark = pytest.mark.gpu
TOL = 2e-5


@pytest.mark.parametrize("name,batch,lr", [("c3a_or50", 3000, 0.1), ("c1b_random", 4096, 0.5),
                                           ("c3a_or50", 70000, 0.05)])
def test_adam_matches_float64_restatement(gpu, name, batch, lr):
    i = load_instance(name)
    P = PortLib()
    b1, b2, eps = 0.9, 0.999, 1e-8
    s = Sampler(DeviceCircuit.from_instance(i),
                SamplerConfig(batch=batch, seed=3, iterations=4, learning_rate=lr, optimizer=Optimizer.ADAM))
    try:
        s.init(1)
        v = s.logits()
        m1 = np.zeros(v.shape, np.float64)
        m2 = np.zeros(v.shape, np.float64)
        for t in range(1, 5):
            tape, _ = P.forward(i, i.cpi, P.embed(v))
            dv, _ = P.backward(i, i.cpi, tape, v)
            g = dv.astype(np.float64)
            m1 = b1 * m1 + (1 - b1) * g
            m2 = b2 * m2 + (1 - b2) * g * g
            want = v.astype(np.float64) - lr * (m1 / (1 - b1 ** t)) / (np.sqrt(m2 / (1 - b2 ** t)) + eps)
            s.step()
            got = s.logits()
            err = np.abs(got.astype(np.float64) - want) / np.maximum(1.0, np.abs(want))
            assert err.max() <= TOL, f"step {t}: max rel err {err.max():.3g}"
            v = got  # continue from the device's V (its f32 rounding)
    finally:
        s.close()


def test_adam_run_emits_valid_unique_solutions(gpu):
    i = load_instance("c3a_or50")
    cfg = SamplerConfig(batch=8192, seed=1, iterations=5, learning_rate=0.2, optimizer=Optimizer.ADAM)
    runs = []
    for _ in range(2):
        s = Sampler(DeviceCircuit.from_instance(i), cfg)
        try:
            st = s.run()
            runs.append((st.unique_count, st.new_unique, s.fetch()))
        finally:
            s.close()
    (u, nu, keys), (u2, nu2, keys2) = runs
    assert u > 0 and u == len(keys)
    assert (u, nu) == (u2, nu2) and np.array_equal(keys, keys2)  # deterministic
    assert verify_keys(i.cnf, keys).all()
    assert len({k.tobytes() for k in keys}) == len(keys)


def test_adam_rejects_bad_hyperparameters(gpu):
    i = load_instance("c3a_or50")
    with pytest.raises(ValueError):
        Sampler(DeviceCircuit.from_instance(i), SamplerConfig(batch=64, optimizer=Optimizer.ADAM, adam_beta1=1.5))
