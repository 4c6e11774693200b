"""The multi-GPU loop below the C-ABI (sgx_run_sharded), on one GPU.

Sample sharding makes the union of N shards at batch B exactly a one-device
run at batch N*B (every random draw is keyed by global row), so each test
runs N ranks -- host threads with the library's in-process exchange, or
processes with torch.distributed (gloo) behind the exchange callbacks -- on
cuda:0 and compares with a single sampler at N*B: global unique count,
per-harvest new-unique trace, attempts, restarts and the solution set.
The NCCL exchange has the same contract (ncclAllGather on the sampler
stream); NCCL needs one GPU per rank, so on a one-GPU box it runs as a world
of one (communicator, collectives and host all-gather all exercised).
"""
import os
import tempfile
import threading

import numpy as np
import pytest

from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig, load_instance,
                                   verify_keys)
from paper_2502_08673_b200 import dist as D

pytestmark = pytest.mark.gpu

CASES = [
    ("c3a_or50", 4096, dict(iterations=3, seed=2)),
    ("c2_iscas", 1024, dict(iterations=2, seed=1)),
    ("mux_chain14", 64, dict(iterations=5, seed=3, max_solutions=1000,
                             restart=RestartPolicy.REINIT_ON_EXHAUST)),
    ("c3a_or50", 2048, dict(iterations=5, seed=4, max_solutions=3000,
                            restart=RestartPolicy.REINIT_ON_EXHAUST)),
    ("c1b_random", 1024, dict(iterations=4, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST,
                              max_restarts=3)),
]


def single(inst, batch, kw):
    s = Sampler(DeviceCircuit.from_instance(inst), SamplerConfig(batch=batch, **kw))
    try:
        st = s.run()
        return st, s.fetch()
    finally:
        s.close()


def as_set(keys):
    return {k.tobytes() for k in keys}


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,batch,kw", CASES, ids=[f"{c[0]}-{c[1]}-{i}" for i, c in enumerate(CASES)])
def test_threads_local_exchange_equal_one_device(gpu, name, batch, kw, world):
    inst = load_instance(name)
    want, want_keys = single(inst, world * batch, kw)
    ex = D.LocalExchanges(world)
    samplers = [Sampler(DeviceCircuit.from_instance(inst), SamplerConfig(batch=batch, row_offset=r * batch, **kw))
                for r in range(world)]
    out, err = [None] * world, [None] * world

    def work(r):
        try:
            out[r] = D.run_native(samplers[r], ex[r])
        except Exception as e:  # noqa: BLE001
            err[r] = e

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    try:
        assert not any(err), err
        keys = [s.fetch() for s in samplers]
    finally:
        for s in samplers:
            s.close()
        ex.close()
    for r in range(world):
        st = out[r]
        assert st.unique_count == want.unique_count
        assert st.new_unique == want.new_unique
        assert st.attempts == want.attempts
        assert st.restarts == want.restarts
    assert sum(len(k) for k in keys) == want.unique_count
    union = set().union(*(as_set(k) for k in keys))
    assert len(union) == want.unique_count
    assert union == as_set(want_keys)
    for k in keys:
        if len(k):
            assert verify_keys(inst.cnf, k).all()


def _proc(rank, world, port, name, batch, kw, outdir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    inst = load_instance(name)
    s = Sampler(DeviceCircuit.from_instance(inst), SamplerConfig(batch=batch, row_offset=rank * batch, **kw))
    ex = D.TorchCallbackExchange(device=0)
    st = D.run_native(s, ex)
    np.save(os.path.join(outdir, f"keys{rank}.npy"), s.fetch())
    with open(os.path.join(outdir, f"stats{rank}.txt"), "w") as f:
        f.write(repr((st.unique_count, st.new_unique, st.attempts, st.restarts)))
    s.close()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,batch,kw", [CASES[0], CASES[3]], ids=["c3a", "c3a-quota"])
def test_processes_torch_exchange_equal_one_device(gpu, name, batch, kw):
    import socket

    import torch.multiprocessing as mp
    world = 2
    inst = load_instance(name)
    want, want_keys = single(inst, world * batch, kw)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    with tempfile.TemporaryDirectory() as d:
        mp.start_processes(_proc, args=(world, port, name, batch, kw, d), nprocs=world, join=True,
                           start_method="spawn")
        keys = [np.load(os.path.join(d, f"keys{r}.npy")) for r in range(world)]
        stats = [eval(open(os.path.join(d, f"stats{r}.txt")).read()) for r in range(world)]
    for st in stats:
        assert st == (want.unique_count, want.new_unique, want.attempts, want.restarts)
    union = set().union(*(as_set(k) for k in keys))
    assert union == as_set(want_keys)


@pytest.mark.parametrize("name,batch,kw", [CASES[1], CASES[3]], ids=["c2", "c3a-quota"])
def test_nccl_exchange_single_rank_equals_sgx_run(gpu, name, batch, kw):
    """The NCCL exchange end to end on the one GPU a box gives: a world of one
    (sgx_nccl_unique_id -> sgx_exchange_nccl_create -> sgx_run_sharded), so the
    communicator set-up, ncclAllGather on the sampler stream and the host
    all-gather all run.  A world of one is exactly sgx_run."""
    inst = load_instance(name)
    want, want_keys = single(inst, batch, kw)
    ex = D.NcclExchange(1, D.nccl_unique_id(), 0, 0)
    s = Sampler(DeviceCircuit.from_instance(inst), SamplerConfig(batch=batch, **kw))
    try:
        st = D.run_native(s, ex)
        keys = s.fetch()
    finally:
        s.close()
        ex.close()
    assert st.unique_count == want.unique_count
    assert st.new_unique == want.new_unique
    assert st.attempts == want.attempts
    assert st.restarts == want.restarts
    assert np.array_equal(keys, want_keys)
