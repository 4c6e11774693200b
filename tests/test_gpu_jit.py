"""GPU parity of the circuit-specialised soft pass (csrc/sgx_jit.cpp).

The kernel is generated per circuit and compiled with NVRTC for sm_100a; it
must reproduce the reference bit for bit exactly like the HBM-tape kernels:
the same golden runs (counts, attempts, new-unique trace, ordered keys), the
same V trajectory as the port oracle's init / embed / forward / backward /
gd_step.  Every test forces the kernel (SoftKernel.JIT: compile at sampler
creation and wait) and asserts that it is the kernel that ran.
"""
import os

import numpy as np
import pytest

from helpers import cfg_kwargs, golden_runs, keys_from_hex, sha
from oracle.oracle import PortLib
from paper_2502_08673_b200 import (DeviceCircuit, Sampler, SamplerConfig, SoftKernel,
                                   load_instance, verify_keys)

pytestmark = pytest.mark.gpu
LOSS_RTOL = 1e-4
SMALL = ("mux_chain14", "c3a_or50", "c1b_random", "c3b_or100", "c1a_planted3sat", "free_inputs",
         "single_model")

_CACHE = {}


def inst(name):
    if name not in _CACHE:
        _CACHE[name] = load_instance(name)
    return _CACHE[name]


def run_jit(i, **kw):
    s = Sampler(DeviceCircuit.from_instance(i), SamplerConfig(soft_kernel=SoftKernel.JIT, **kw))
    try:
        st = s.run()
        keys = s.fetch()
        info = s.soft_info()
    finally:
        s.close()
    return st, keys, info


@pytest.mark.parametrize("rec", [r for r in golden_runs() if r["instance"] in SMALL],
                         ids=lambda r: f"{r['instance']}-{r['config']}")
def test_jit_runs_match_reference(gpu, rec):
    i = inst(rec["instance"])
    st, keys, info = run_jit(i, **cfg_kwargs(rec["config"]))
    assert st.unique_count == rec["unique"]
    assert st.attempts == rec["attempts"]
    assert st.restarts == rec["restarts"]
    assert st.new_unique == rec["new_unique"]
    np.testing.assert_allclose(st.loss_trace, rec["loss_trace"], rtol=LOSS_RTOL, atol=0)
    assert sha(keys) == rec["keys_sha256"]
    if rec.get("keys"):
        assert np.array_equal(keys, keys_from_hex(rec["keys"]))
    if len(keys):
        assert verify_keys(i.cnf, keys).all()
    if st.loss_trace:  # at least one step ran: it must have been the specialised kernel
        assert info["jit_state"] == "ready", info
        assert info["last"] == "jit" and info["jit_steps"] > 0, info


@pytest.mark.parametrize("name,batch", [("c3a_or50", 3000), ("c3a_or50", 1 << 16), ("c3b_or100", 65536),
                                        ("c1b_random", 5000), ("c1a_planted3sat", 2048),
                                        ("mux_chain14", 70000)])
def test_jit_logit_trajectory_bit_exact(gpu, name, batch):
    """V after each specialised step equals the port oracle's init_soft_inputs,
    embed, forward, backward and gd_step bit for bit (vec 1/2/4 layouts)."""
    i = inst(name)
    P = PortLib()
    s = Sampler(DeviceCircuit.from_instance(i),
                SamplerConfig(batch=batch, seed=3, iterations=3, soft_kernel=SoftKernel.JIT))
    try:
        s.init(1)
        v = P.init_soft_inputs(batch, len(i.cpi), 3, 1).astype(np.float32)
        for _ in range(3):
            s.step()
            tape, _ = P.forward(i, i.cpi, P.embed(v))
            dv, _ = P.backward(i, i.cpi, tape, v)
            v = (v - np.float32(10.0) * dv).astype(np.float32)
            got = s.logits()
            bad = np.nonzero(got.view(np.uint32) != v.view(np.uint32))
            assert bad[0].size == 0, f"{bad[0].size} logits differ, first at row {bad[0][0]} col {bad[1][0]}"
        info = s.soft_info()
        assert info["last"] == "jit" and info["jit_steps"] == 3, info
    finally:
        s.close()


def test_jit_and_hbm_kernels_agree_at_bench_batch(gpu):
    """C3a at the bench batch (2^20 rows): the specialised kernel and the
    HBM-tape kernels give the same run (counts, trace, ordered keys)."""
    i = inst("c3a_or50")
    kw = dict(batch=1 << 20, iterations=2, seed=1)
    st_j, k_j, info = run_jit(i, **kw)
    assert info["last"] == "jit"
    s = Sampler(DeviceCircuit.from_instance(i), SamplerConfig(soft_kernel=SoftKernel.HBM, **kw))
    try:
        st_h = s.run()
        k_h = s.fetch()
        assert s.soft_info()["last"] == "hbm"
    finally:
        s.close()
    assert st_j.new_unique == st_h.new_unique
    assert st_j.loss_trace == st_h.loss_trace
    assert np.array_equal(k_j, k_h)


def test_process_exits_cleanly_with_a_compile_in_flight(gpu):
    """A short process whose AUTO soft pass started a background NVRTC compile
    exits with status 0 (the compile is joined before teardown: the Python
    package's atexit -> sgx_jit_quiesce, and the library's own atexit)."""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for batch in ("4096", "1048576"):
        r = subprocess.run([sys.executable, os.path.join(root, "tools", "exit_probe.py"), "c3a_or50", batch, "1"],
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, (batch, r.returncode, r.stderr[-2000:])
        assert "done 1000" in r.stdout
