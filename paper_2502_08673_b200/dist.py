"""Multi-GPU sampling: sample sharding with a per-harvest fingerprint exchange.

The reference is one process; rows are independent
and every random draw is keyed by (seed, restart, [iter,] row, col)
(sampler.cpp:54-64, :132-137).  So rank g of N samples global rows
[g*B, (g+1)*B) with cfg.row_offset = g*B, and the union of the shards is
exactly a one-device run at batch N*B.  The only data-path collective is the
all-gather of each harvest's new 64-bit solution fingerprints (NCCL over
NVLink when the group is NCCL), which keeps uniqueness global: a solution
found by several ranks in the same harvest counts once, for the lowest rank
(the reference's row order), and every rank's table learns every
fingerprint.  Quota, "restart found nothing" and timeout decisions use
all-gathered counters so every rank takes the same branch (run_impl,
sampler.cpp:89-194, restated over the union).

``run_sharded`` is written against two small interfaces so its control flow
can be exercised on CPU (gloo) with a stand-in sampler:
  * a sampler with init(restart) / step() / harvest_local(restart, it) ->
    (n_new, fps) / harvest_merge(gathered, counts, world, rank) -> n_won /
    harvest_commit(quota_left) -> (attempts, added); optionally
    step_async() -> slot / step_loss(slot) (the next step then samples while
    the harvest's exchange is in flight) and gather_stride / counts(gathered,
    world) (the counts ride in the fingerprint all-gather);
  * an exchange with all_gather_int(x) -> list[int] and
    all_gather_fps(fps, stride) -> gathered.
Per harvest on the device path: one all-gather of fingerprints + counts, one
of the merged counts (plus one of attempts only under a quota).
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

from . import _lib


class _DevArray:
    """Zero-copy view of a library-owned device buffer for torch."""

    def __init__(self, ptr: int, n: int, device: int):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                         "version": 3}


class DeviceShard:
    """A Sampler driven through the split harvest of the C-ABI."""

    def __init__(self, sampler):
        self.s = sampler
        self.L = _lib.load()
        self.stride = int(self.L.sgx_fingerprint_stride(sampler.h))
        self.gather_stride = self.stride + 1  # fingerprints, then their count
        self.device = sampler.dc.device

    def init(self, restart: int):
        self.s.init(restart)

    def step(self) -> float:
        return self.s.step()

    def step_async(self) -> int:
        slot = C.c_int32()
        _lib.check(self.L.sgx_step_async(self.s.h, C.byref(slot)))
        return slot.value

    def step_loss(self, slot: int) -> float:
        x = C.c_double()
        _lib.check(self.L.sgx_step_loss(self.s.h, slot, C.byref(x)))
        return x.value

    def counts(self, gathered, world: int) -> list[int]:
        return [int(v) for v in gathered.view(world, self.gather_stride)[:, self.stride].cpu()]

    def harvest_local(self, restart: int, it: int):
        import torch
        n = C.c_int64()
        ptr = C.c_void_p()
        _lib.check(self.L.sgx_harvest_local(self.s.h, restart, it, C.byref(n), C.byref(ptr)))
        fps = torch.as_tensor(_DevArray(ptr.value, self.gather_stride, self.device),
                              device=f"cuda:{self.device}")
        return n.value, fps

    def harvest_merge(self, gathered, counts, world: int, rank: int) -> int:
        import numpy as np
        won = C.c_int64()
        cnt = np.ascontiguousarray(counts, np.int64)
        _lib.check(self.L.sgx_harvest_merge(self.s.h, C.c_void_p(gathered.data_ptr()),
                                            _lib.ptr(cnt, C.c_int64), world, rank, self.gather_stride,
                                            C.byref(won)))
        return won.value

    def harvest_commit(self, quota_left: int):
        att, add = C.c_int64(), C.c_int64()
        _lib.check(self.L.sgx_harvest_commit(self.s.h, quota_left, C.byref(att), C.byref(add)))
        return att.value, add.value


class TorchExchange:
    """torch.distributed collectives (NCCL on GPU tensors, gloo on CPU)."""

    def __init__(self, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.device = torch.device(device) if device is not None else torch.device("cpu")
        self.torch = torch
        # gloo moves host tensors only: device payloads are staged through the
        # host (a test set-up: several ranks on one GPU, where NCCL refuses)
        self.host_staged = dist.get_backend(group) == "gloo"
        self.coll_device = torch.device("cpu") if self.host_staged else self.device

    def all_gather_int(self, x: int) -> list[int]:
        t = self.torch.tensor([int(x)], dtype=self.torch.int64, device=self.coll_device)
        out = self.torch.zeros(self.world, dtype=self.torch.int64, device=self.coll_device)
        self.dist.all_gather_into_tensor(out, t, group=self.group)
        return [int(v) for v in out.cpu()]

    def all_gather_fps(self, fps, stride: int):
        src = fps[:stride].contiguous()
        if self.host_staged:
            src = src.cpu()
        out = self.torch.empty(self.world * stride, dtype=self.torch.int64, device=src.device)
        self.dist.all_gather_into_tensor(out, src, group=self.group)
        if self.host_staged and fps.is_cuda:
            out = out.to(fps.device)
        if out.is_cuda:
            self.torch.cuda.current_stream(out.device).synchronize()
        return out


@dataclass
class ShardStats:
    unique_count: int = 0           # global unique solutions (all ranks)
    local_count: int = 0            # solutions this rank holds
    attempts: int = 0               # global rows pushed through verification
    restarts: int = 0
    timed_out: bool = False
    loss_trace: list = field(default_factory=list)   # this rank's mean loss per step
    new_unique: list = field(default_factory=list)   # global new per harvest
    wall_time_s: float = 0.0


def run_sharded(shard, ex, cfg, rank: int, world: int, stride: int) -> ShardStats:
    """run_impl (sampler.cpp:89-194) over the union of `world` shards."""
    if int(cfg.restart) in (2, 3):
        raise ValueError("RestartPolicy.REINIT_ROWS / REINIT_INVALID are single-device only (sgx_run)")
    st = ShardStats()
    t0 = time.perf_counter()
    quota = cfg.max_solutions > 0

    def quota_met():
        return quota and st.unique_count >= cfg.max_solutions

    def out_of_time():
        # every rank must take the same branch: any rank over time stops all
        late = cfg.timeout_s > 0 and time.perf_counter() - t0 >= cfg.timeout_s
        return max(ex.all_gather_int(1 if late else 0)) > 0 if cfg.timeout_s > 0 else False

    overlap = hasattr(shard, "step_async")
    gstride = getattr(shard, "gather_stride", stride)

    def harvest(restart, it, launch_next):
        """One harvest over the union; with launch_next the next step is
        launched as soon as the local harvest kernels are done (it only reads
        V; the backward waits for the harvest's reads on the device)."""
        n_new, fps = shard.harvest_local(restart, it)
        slot = shard.step_async() if launch_next else None
        gathered = ex.all_gather_fps(fps, gstride)
        counts = shard.counts(gathered, world) if hasattr(shard, "counts") else ex.all_gather_int(n_new)
        won = shard.harvest_merge(gathered, counts, world, rank)
        wons = ex.all_gather_int(won)
        left = cfg.max_solutions - st.unique_count if quota else None
        before = sum(wons[:rank])
        my_left = max(0, left - before) if quota else -1
        att, add = shard.harvest_commit(my_left)
        if quota and my_left == 0:
            att = 0  # a lower rank filled the quota: these rows come after the cut
        # global accepted, in rank order (identical on every rank)
        acc = 0
        for w in wons:
            take = w if not quota else max(0, min(w, left - acc))
            acc += take
        st.unique_count += acc
        st.local_count += add
        # without a quota every rank attempts its whole batch
        st.attempts += sum(ex.all_gather_int(att)) if quota else att * world
        st.new_unique.append(acc)
        return slot

    def speculate(it):  # the reference runs step `it` unless quota or time stop it first
        return overlap and not quota and cfg.timeout_s <= 0 and it <= cfg.iterations

    restart = 0
    while True:
        shard.init(restart)
        before = st.unique_count
        slot = harvest(restart, 0, speculate(1))
        for it in range(1, cfg.iterations + 1):
            if quota_met():
                break
            if out_of_time():
                st.timed_out = True
                break
            if overlap:
                if slot is None:
                    slot = shard.step_async()
                loss = shard.step_loss(slot)
            else:
                loss = shard.step()
            st.loss_trace.append(loss / cfg.batch)
            slot = harvest(restart, it, speculate(it + 1))
        if quota_met() or st.timed_out:
            break
        if int(cfg.restart) != 1:
            break
        if st.unique_count == before:
            break
        if restart >= (cfg.max_restarts if cfg.max_restarts > 0 else 1000):
            break
        if out_of_time():
            st.timed_out = True
            break
        st.restarts = restart + 1
        restart += 1
    st.wall_time_s = time.perf_counter() - t0
    return st


# --------------------------------------------------------------- native loop
# sgx_run_sharded: the same protocol in C++ below the C-ABI (one all-gather
# of fingerprints per harvest; the union's size is derived locally).  Python
# only supplies the collective: the library's NCCL exchange (one process per
# GPU), its in-process exchange (one thread per rank), or torch.distributed
# through callbacks (gloo, host-staged: several ranks on one GPU in tests).

def nccl_unique_id() -> bytes:
    L = _lib.load()
    buf = C.create_string_buffer(128)
    _lib.check(L.sgx_nccl_unique_id(buf))
    return buf.raw


class NcclExchange:
    """The library's NCCL communicator (ncclAllGather on the sampler stream)."""

    def __init__(self, world: int, uid: bytes, rank: int, device: int):
        self.L = _lib.load()
        self.ex = _lib.Exchange()
        _lib.check(self.L.sgx_exchange_nccl_create(world, uid, rank, device, C.byref(self.ex)))

    def close(self):
        if self.ex.user:
            _lib.check(self.L.sgx_exchange_nccl_destroy(C.byref(self.ex)))


class LocalExchanges:
    """In-process group: exchanges[r] for the host thread running rank r."""

    def __init__(self, world: int):
        self.L = _lib.load()
        self.arr = (_lib.Exchange * world)()
        _lib.check(self.L.sgx_exchange_local_create(world, self.arr))

    def __getitem__(self, r):
        return self.arr[r]

    def close(self):
        if self.arr[0].user:
            _lib.check(self.L.sgx_exchange_local_destroy(C.byref(self.arr[0])))


class TorchCallbackExchange:
    """torch.distributed collectives behind the C callbacks.  With gloo the
    device payload is staged through host memory (the sampler stream is
    synchronised first, and recv is written before returning)."""

    def __init__(self, device: int, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.device = device
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.host_staged = dist.get_backend(group) == "gloo"
        self._dev = _lib.ALLGATHER_DEVICE(self._allgather_device)
        self._host = _lib.ALLGATHER_HOST(self._allgather_host)
        self.ex = _lib.Exchange(None, self.rank, self.world, self._dev, self._host)

    def _view(self, ptr, nbytes):
        t = self.torch
        arr = _DevArray(ptr, nbytes // 8, self.device)
        return t.as_tensor(arr, device=f"cuda:{self.device}")

    def _allgather_device(self, user, send, recv, nbytes, stream):
        try:
            t = self.torch
            t.cuda.ExternalStream(stream, device=f"cuda:{self.device}").synchronize()
            src = self._view(send, nbytes)
            dst = self._view(recv, nbytes * self.world)
            if self.host_staged:
                out = t.empty(self.world * (nbytes // 8), dtype=t.int64)
                self.dist.all_gather_into_tensor(out, src.cpu(), group=self.group)
                dst.copy_(out)
            else:
                self.dist.all_gather_into_tensor(dst, src.clone(), group=self.group)
            t.cuda.synchronize(self.device)
            return 0
        except Exception as e:  # noqa: BLE001 -- reported through the status code
            print(f"allgather_device failed: {e!r}", flush=True)
            return -1

    def _allgather_host(self, user, send, recv, n):
        try:
            t = self.torch
            x = t.tensor([send[i] for i in range(n)], dtype=t.int64)
            dev = "cpu" if self.host_staged else f"cuda:{self.device}"
            out = t.empty(self.world * n, dtype=t.int64, device=dev)
            self.dist.all_gather_into_tensor(out, x.to(dev), group=self.group)
            for i, v in enumerate(out.cpu().tolist()):
                recv[i] = v
            return 0
        except Exception as e:  # noqa: BLE001
            print(f"allgather_host failed: {e!r}", flush=True)
            return -1

    def close(self):
        pass


def run_native(sampler, ex) -> ShardStats:
    """sgx_run_sharded on this rank's sampler; ex is an _lib.Exchange or one
    of the wrappers above.  Returns the global statistics."""
    import numpy as np
    L = _lib.load()
    exs = ex.ex if hasattr(ex, "ex") else ex
    st = _lib.RunStatsC()
    _lib.check(L.sgx_run_sharded(sampler.h, C.byref(exs), C.byref(st)))
    loss = np.zeros(max(1, st.n_loss), np.float64)
    nu = np.zeros(max(1, st.n_harvest), np.int64)
    _lib.check(L.sgx_run_traces(sampler.h, _lib.ptr(loss, C.c_double), _lib.ptr(nu, C.c_int64)))
    return ShardStats(unique_count=st.unique_count, local_count=int(L.sgx_solution_count(sampler.h)),
                      attempts=st.attempts, restarts=st.restarts, timed_out=bool(st.timed_out),
                      loss_trace=[float(x) for x in loss[:st.n_loss]],
                      new_unique=[int(x) for x in nu[:st.n_harvest]], wall_time_s=st.wall_time_s)
