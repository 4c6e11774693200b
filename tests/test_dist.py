"""Multi-process control flow of the sharded sampler (paper_2502_08673_b200/dist.py).

CPU (gloo, world_size 2): run_sharded drives a stand-in shard whose rows
produce deterministic fingerprints keyed by (restart, iter, GLOBAL row) -- the
same keying the device uses -- so the union of the two shards must behave
exactly like one process holding both row ranges: identical global unique
counts per harvest, quota cut at the same solution, identical restart count.
The device half of the protocol (split harvest through the C-ABI) is checked
on the GPU in tests/test_gpu_dist.py.
"""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_08673_b200 import RestartPolicy, SamplerConfig
from paper_2502_08673_b200.dist import TorchExchange, run_sharded


def _fp(restart, it, row):
    # a few hundred distinct "solutions", heavily repeated across rows,
    # exhausted after a handful of restarts
    x = (restart * 7919 + it * 104729 + row * 31) % 97 + (restart % 3) * 97
    return x * 0x9E3779B97F4A7C15 % (1 << 63) + 1


class FakeShard:
    """Rows [offset, offset+B): row r is valid iff (r + it) % 3 != 0."""

    def __init__(self, batch, offset):
        self.B, self.off = batch, offset
        self.table = set()

    def init(self, restart):
        pass

    def step(self):
        return 1.0 * self.B

    def harvest_local(self, restart, it):
        self.new_rows, seen = [], set()
        for r in range(self.off, self.off + self.B):
            if (r + it) % 3 == 0:
                continue
            fp = _fp(restart, it, r)
            if fp not in self.table and fp not in seen:
                seen.add(fp)
                self.new_rows.append(fp)
        self.table |= seen
        return len(self.new_rows), np.array(self.new_rows, np.int64)

    def harvest_merge(self, gathered, counts, world, rank):
        lower = set()
        for g in range(rank):
            lower |= set(gathered[g][:counts[g]].tolist())
        for g in range(world):
            self.table |= set(gathered[g][:counts[g]].tolist())
        self.won = [fp for fp in self.new_rows if fp not in lower]
        return len(self.won)

    def harvest_commit(self, quota_left):
        take = self.won if quota_left < 0 else self.won[:quota_left]
        return self.B, len(take)


class ListExchange:
    """all_gather of fingerprint lists over a gloo group."""

    def __init__(self, ex):
        self.ex = ex

    def all_gather_int(self, x):
        return self.ex.all_gather_int(x)

    def all_gather_fps(self, fps, stride):
        out = [None] * self.ex.world
        dist.all_gather_object(out, fps)
        return out


def _worker(rank, world, port, cfg, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = FakeShard(cfg.batch, rank * cfg.batch)
        st = run_sharded(shard, ListExchange(TorchExchange()), cfg, rank, world, cfg.batch)
        q.put((rank, st.unique_count, st.new_unique, st.restarts, st.attempts))
    finally:
        dist.destroy_process_group()


def _single(cfg, world):
    """The same control flow in one process over all rows (reference order)."""
    shard = FakeShard(cfg.batch * world, 0)

    class Solo:
        world = 1

        def all_gather_int(self, x):
            return [x]

        def all_gather_fps(self, fps, stride):
            return [fps]

    big = SamplerConfig(**{**cfg.__dict__, "batch": cfg.batch * world})
    return run_sharded(shard, Solo(), big, 0, 1, big.batch)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("cfg", [
    SamplerConfig(batch=40, iterations=3, seed=1),
    SamplerConfig(batch=40, iterations=2, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST),
    SamplerConfig(batch=40, iterations=3, seed=1, max_solutions=57),
    SamplerConfig(batch=25, iterations=2, seed=1, max_solutions=130,
                  restart=RestartPolicy.REINIT_ON_EXHAUST),
])
def test_two_ranks_equal_one_process(cfg):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _single(cfg, world)
    for rank, uniq, nu, restarts, attempts in res:
        assert uniq == want.unique_count
        assert nu == want.new_unique
        assert restarts == want.restarts
    if cfg.max_solutions:
        assert res[0][1] == cfg.max_solutions


# ---------------------------------------------------------------------------
# C5 sweep driver (paper_2502_08673_b200/sweep.py) at world size 2: every
# suite instance goes through run_sharded; both ranks must report the same
# per-instance global counts as one process over the union, and the same
# family summary.

SUITE = ["c5/or50_01", "c5/q_17", "c5/s15850_33", "c5/prod_45", "c5/blasted200_55"]


def _suite_runner(solo):
    from paper_2502_08673_b200.sweep import family

    def run_one(name, batch, rank, world):
        b = 24 + 7 * SUITE.index(name)  # small stand-in batch per instance
        cfg = SamplerConfig(batch=b, iterations=2, seed=1)
        if solo:
            st = _single(cfg, world)
        else:
            shard = FakeShard(b, rank * b)
            st = run_sharded(shard, ListExchange(TorchExchange()), cfg, rank, world, b)
        return st.unique_count, 0.5 + rank + len(family(name))

    return run_one


def _suite_worker(rank, world, port, q):
    from paper_2502_08673_b200.sweep import run_suite, summarize
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch

        def sync(x):
            t = torch.tensor([x], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return float(t.item())
        res = run_suite(SUITE, _suite_runner(False), rank, world, sync)
        q.put((rank, [(r.name, r.unique, r.seconds) for r in res], summarize(res, world)))
    finally:
        dist.destroy_process_group()


def test_c5_suite_two_ranks_equal_one_process():
    from paper_2502_08673_b200.sweep import FAMILY_BATCH, run_suite, summarize
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_suite_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = run_suite(SUITE, _suite_runner(True), 0, world)
    for rank, rows, summ in got:
        assert [(n, u) for n, u, _ in rows] == [(r.name, r.unique) for r in want]
        # device time is the max over ranks (rank 1's stand-in time here)
        assert [s for _, _, s in rows] == [r.seconds + 1 for r in want]
        assert summ == got[0][2]
        assert summ["unique"] == sum(r.unique for r in want)
        assert set(summ["families"]) == {"or", "q", "s15850", "prod", "blasted"}
        assert all(f["batch_per_gpu"] == FAMILY_BATCH[k] for k, f in summ["families"].items())
    assert summarize(want, 1)["unique"] == got[0][2]["unique"]


def test_reinit_rows_policy_is_single_device_only():
    from paper_2502_08673_b200 import RestartPolicy, SamplerConfig
    from paper_2502_08673_b200.dist import run_sharded
    with pytest.raises(ValueError):
        run_sharded(None, None, SamplerConfig(restart=RestartPolicy.REINIT_ROWS), 0, 1, 1024)
