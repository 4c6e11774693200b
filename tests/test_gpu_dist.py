"""GPU: the split harvest (sgx_harvest_local / merge / commit) across shards.

Two shards (global rows [0, B) and [B, 2B)) run in lock-step in two threads
on one GPU with an in-process exchange; their union must reproduce a single
sampler at batch 2B exactly: the same global new-unique count per harvest and
the same solution set (first-row-wins dedup across shards = reference row
order), with and without a quota.
"""
import threading

import numpy as np
import pytest

from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig,
                                   load_instance, run_instance, verify_keys)
from paper_2502_08673_b200.dist import DeviceShard, run_sharded

pytestmark = pytest.mark.gpu


class ThreadExchange:
    def __init__(self, world):
        self.world = world
        self.bar = threading.Barrier(world, timeout=120)  # a failing rank must not hang the other
        self.slots = [None] * world

    def view(self, rank):
        ex = self

        class V:
            def all_gather_int(self, x):
                ex.slots[rank] = x
                ex.bar.wait()
                out = list(ex.slots)
                ex.bar.wait()
                return out

            def all_gather_fps(self, fps, stride):
                import torch
                ex.slots[rank] = fps[:stride].clone()
                torch.cuda.current_stream().synchronize()
                ex.bar.wait()
                out = torch.cat(list(ex.slots))
                torch.cuda.current_stream().synchronize()  # the library runs on its own stream
                ex.bar.wait()
                return out
        return V()


def run_two_shards(inst, cfg):
    world = 2
    dc = DeviceCircuit.from_instance(inst)
    ex = ThreadExchange(world)
    shards, out = [], [None] * world
    for r in range(world):
        c = SamplerConfig(**{**cfg.__dict__, "row_offset": r * cfg.batch})
        shards.append(DeviceShard(Sampler(dc, c)))

    def work(r):
        out[r] = run_sharded(shards[r], ex.view(r), cfg, r, world, shards[r].stride)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    keys = [s.s.fetch() for s in shards]
    return out, keys


@pytest.mark.parametrize("name,cfg", [
    ("c3a_or50", SamplerConfig(batch=3000, iterations=3, seed=4)),
    ("c3a_or50", SamplerConfig(batch=3000, iterations=3, seed=4, max_solutions=2500)),
    ("c1b_random", SamplerConfig(batch=700, iterations=2, seed=2, max_solutions=100000,
                                 restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=3)),
    ("c2_iscas", SamplerConfig(batch=1024, iterations=1, seed=1)),
])
def test_two_shards_equal_one_sampler(gpu, name, cfg):
    inst = load_instance(name)
    stats, keys = run_two_shards(inst, cfg)
    big = SamplerConfig(**{**cfg.__dict__, "batch": 2 * cfg.batch})
    want = run_instance(inst, big)
    for st in stats:
        assert st.unique_count == want.stats.unique_count
        assert st.new_unique == want.stats.new_unique
        assert st.restarts == want.stats.restarts
    union = np.concatenate(keys)
    assert len(union) == want.stats.unique_count
    assert {k.tobytes() for k in union} == {k.tobytes() for k in want.solutions.keys}
    assert verify_keys(inst.cnf, union).all()
