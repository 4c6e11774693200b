#!/usr/bin/env python
"""Benchmark: unique valid SAT solutions per second (BASELINE.json metric).

Workload (default, the largest single-GPU config, BASELINE configs[3] /
SURVEY.md section 8 "C4"): the blasted_case-shaped synthetic CNF
encode(random_circuit(31337, 400, 400, 100, 2)) -- 40,400 vars, 132,151
clauses, an 88,866-node circuit 877 levels deep -- sampled at batch 65,536
rows per GPU with the reference hyper-parameters (GD, lr 10, 5 iterations,
seed 1, f32).  --workload c2_iscas is configs[1] (ISCAS89-shaped), c3a_or50
the or-50 shape of the time-to-1k metric.

One "step" = one restart of satgrad::run: init_soft_inputs, the iteration-0
harvest, then 5 x (embed+forward+loss+backward+GD, harvest) over the whole
batch.  K steps run back to back inside one sgx_run (ReinitOnExhaust with a
restart budget of K), W warm-up restarts before.  Inputs (C4 tape 17.4 GB,
C2 3.5 GB) exceed the 126 MB L2, so no explicit flush is needed between steps.

  value   unique solutions found in the timed restarts / device time
          (CUDA events on the sampler stream, max over ranks)
  e2e     the same metric through the public API run() from host buffers:
          circuit upload (H2D), the run, and fetching every solution key (D2H)
  invalid solutions among the e2e result that fail the CNF, are malformed or
          repeat (device re-verification after the timed region)
  --impl reference   the reference's own CPU sampler (oracle/_ref, built from
          /root/reference sources) on every host core, at the SAME workload,
          batch and hyper-parameters, bounded by the reference's own
          timeout_s.

Multi-GPU (torchrun): rank g samples global rows [g*B, (g+1)*B) (RNG keyed by
global row, so shards are disjoint slices of one big batch); solutions are
deduplicated across ranks by an all-gather of 64-bit fingerprints.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "unique valid solutions/sec"
UNIT = "solutions/s"
WORKLOADS = {
    # name: (instance file, default batch, cpu_baseline sample batch)
    "c4_blasted": ("c4_blasted", 65536, 512),
    "c2_iscas": ("c2_iscas", 65536, 2048),
    "c3a_or50": ("c3a_or50", 1 << 20, 20000),
    "c3b_or100": ("c3b_or100", 1 << 20, 20000),
    "c1b_random": ("c1b_random", 1024, 1024),
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.samples = []
        self.start = 0
        self.proc = None
        self.thread = None

    def __enter__(self):
        if os.environ.get("BENCH_NOCLOCK"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "25"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi's start-up (NVML init) stalls the driver for a while:
            # let it finish before the timed region, on its first sample.
            t0 = time.perf_counter()
            while not self.samples and time.perf_counter() - t0 < 5.0:
                time.sleep(0.02)
            time.sleep(0.3)
            self.start = len(self.samples)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            if self.thread:
                self.thread.join(timeout=2)

    def summary(self):
        during = self.samples[self.start:]
        used, pre = during, False
        if not during and self.samples:  # region shorter than one poll: the sample just before it
            used, pre = self.samples[-1:], True
        if not used:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(s[1]) for s in used if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in used if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in used for i in range(4)
                          if s[5 + i].lower().startswith("active")})
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
               "samples": len(during), "poll_ms": 25}
        if pre:
            out["from_sample_before_region"] = True
        return out


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        # BENCH_DIST_BACKEND=gloo: a test set-up running several ranks on fewer
        # GPUs (payloads staged through the host); the bench itself uses NCCL.
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl")
        if args.impl != "reference":
            local = local % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local)
        dist.init_process_group(backend if args.impl != "reference" else "gloo")
        pg = dist
    return world, rank, local, pg


def cpu_reference(inst_name, batch, iterations, seed, steps=1, timeout_s=0.0, f32=True):
    """The reference's satgrad::run on the host cores (oracle/_ref); falls back
    to the C port (oracle/libsgx_oracle.so) when the reference was not built."""
    from paper_2502_08673_b200 import load_instance, write_dimacs
    from oracle.oracle import PortLib, RefInstance, ref_available
    cores = os.cpu_count() or 1
    inst = load_instance(inst_name)
    uniq, wall, timed_out, attempts, new_unique = 0, 0.0, False, 0, []
    if ref_available():
        ri = RefInstance.from_dimacs(write_dimacs(inst.cnf))
        kind = "reference"
        for _ in range(steps):
            r = ri.run(batch=batch, iterations=iterations, seed=seed, threads=cores,
                       use_f32=f32, timeout_s=timeout_s)
            uniq += r.unique
            wall += r.wall
            timed_out |= r.timed_out
            attempts += r.attempts
            new_unique += r.new_unique
    else:
        kind, cores = "port", 1
        for _ in range(steps):
            r = PortLib().run(inst, batch=batch, iterations=iterations, seed=seed,
                              timeout_s=timeout_s)
            uniq += r.unique
            wall += r.wall
            timed_out |= r.timed_out
            attempts += r.attempts
            new_unique += r.new_unique
    tmo = f", timeout_s={timeout_s:g}" if timeout_s > 0 else ""
    return {"value": uniq / wall if wall > 0 else 0.0, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{steps} x satgrad::run(batch={batch}, iterations={iterations}, seed={seed}, "
                      f"{'f32' if f32 else 'f64'}, threads={cores}{tmo}) on {inst_name}: {uniq} unique "
                      f"in {wall:.2f} s" + (" (stopped by the timeout)" if timed_out else ""),
            "unique": uniq, "wall_s": wall, "timed_out": timed_out, "attempts": attempts,
            "new_unique": new_unique}


def time_to_1k(dev, with_cpu=True, name="c3a_or50", batch=1 << 20):
    """BASELINE.json's second metric: time to 1,000 unique valid solutions on
    the or-50 shape at a 1M-row batch (quota 1000, ReinitOnExhaust, as the
    reference's `bench` subcommand runs it, satgrad_main.cpp:319-327)."""
    from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig,
                                       load_instance, run_instance)
    inst = load_instance(name)
    cfg = SamplerConfig(batch=batch, iterations=5, seed=1, max_solutions=1000,
                        restart=RestartPolicy.REINIT_ON_EXHAUST)
    dc = DeviceCircuit.from_instance(inst, device=dev)
    s = Sampler(dc, cfg)
    s.run()  # warm-up
    from paper_2502_08673_b200 import jit_quiesce
    jit_quiesce()  # the specialised soft pass compiled (once per process), as in the main measurement
    dev_ms = []
    for _ in range(5):
        st = s.run()
        assert st.unique_count == 1000
        dev_ms.append(st.device_ms)
    s.close()
    run_instance(inst, cfg, device=dev)  # warm-up of the public path (pool, host mapping)
    e2e = []
    for _ in range(5):  # a ~1.5 ms latency: the median of 5 calls
        t0 = time.perf_counter()
        res = run_instance(inst, cfg, device=dev)  # public API: upload, run, fetch
        e2e.append(1000.0 * (time.perf_counter() - t0))
        assert res.stats.unique_count == 1000
    e2e_ms = statistics.median(e2e)
    out = {"workload": name, "batch": batch, "quota": 1000,
           "device_ms": statistics.median(dev_ms), "e2e_ms": e2e_ms,
           "e2e_ms_min_max": [min(e2e), max(e2e)], "unique": res.stats.unique_count}
    if with_cpu:
        from paper_2502_08673_b200 import write_dimacs
        from oracle.oracle import RefInstance, ref_available
        if ref_available():
            ri = RefInstance.from_dimacs(write_dimacs(inst.cnf))
            r = ri.run(batch=batch, iterations=5, seed=1, max_solutions=1000, restart=True,
                       threads=os.cpu_count() or 1, use_f32=True)
            out["cpu_reference_s"] = r.wall
            out["cpu_cores"] = os.cpu_count()
            out["speedup_e2e"] = r.wall / (e2e_ms / 1000.0)
    return out


def run_reference_arm(args, world, rank):
    """The reference's satgrad::run on this box's host cores at the SAME
    config as the B200 arm (workload, batch, iterations, lr, seed, f32).  One
    run of the whole batch is minutes of CPU work (its harvest is single
    threaded), so the K timed steps share ONE run bounded by
    the reference's own timeout_s (checked before each iteration,
    sampler.cpp:164-168), as SURVEY.md 8(d) prescribes; W warm-up steps are a
    small run that pages the library and instance in."""
    name, batch, sample_batch = WORKLOADS[args.workload]
    batch = args.batch or batch
    if rank != 0:
        return
    if args.warmup > 0:
        cpu_reference(name, 256, 1, 1, steps=1)
    budget = float(os.environ.get("BENCH_REF_TIMEOUT", "120"))
    res = cpu_reference(name, batch, args.iterations, 1, steps=1, timeout_s=budget)
    line = {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * res["wall_s"] / max(1, args.steps), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": name, "batch": batch, "global_batch": batch * world,
                   "iterations": args.iterations, "lr": 10.0, "seed": 1},
        "reference_run": {"runs": 1, "timeout_s": budget, "timed_out": res["timed_out"],
                          "attempts": res["attempts"], "new_unique": res["new_unique"],
                          "wall_s": res["wall_s"],
                          "note": "the K steps share one timeout-bounded satgrad::run of the full batch; "
                                  "ms_per_step = its wall / K"},
        "cpu_baseline": {k: res[k] for k in ("value", "unit", "cores", "kind", "sample")},
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_b200_arm(args, world, rank, local, dist):
    import torch
    from paper_2502_08673_b200 import (DeviceCircuit, RestartPolicy, Sampler, SamplerConfig,
                                       load_instance, run_instance)
    name, batch, ref_batch = WORKLOADS[args.workload]
    batch = args.batch or batch
    dev = local
    torch.cuda.set_device(dev)
    # max-over-ranks reductions: on the device over NCCL, on the host over gloo
    coll_dev = "cpu" if (dist and dist.get_backend() == "gloo") else f"cuda:{dev}"
    inst = load_instance(name)
    dc = DeviceCircuit.from_instance(inst, device=dev)
    info = dc.info()

    def cfg_for(restarts):
        # Presize the solution store / table for the run's upper bound (every
        # harvested row unique), so no growth lands inside the timed region.
        # (sized from the timed run for the warm-up too, so the timed sampler
        # reuses the warm-up's pool memory instead of mapping fresh pages).
        # (+2 batches: the store grows ahead once fewer than a batch of rows
        # are left, sgx_api.cpp harvest_back_finish)
        cap = (max(1, args.steps) * (args.iterations + 1) + 2) * batch * world
        return SamplerConfig(batch=batch, iterations=args.iterations, seed=1,
                             restart=RestartPolicy.REINIT_ON_EXHAUST if restarts > 1 else
                             RestartPolicy.NONE, max_restarts=max(1, restarts - 1),
                             row_offset=rank * batch, solution_capacity=cap)

    ex = None
    if world > 1:
        from paper_2502_08673_b200 import dist as D
        if dist.get_backend() == "gloo":  # test set-up: ranks share GPUs, payloads via the host
            ex = D.TorchCallbackExchange(device=dev)
        else:  # the library's own NCCL communicator (id from rank 0)
            uid = [D.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            ex = D.NcclExchange(world, uid[0], rank, dev)
    sampler = Sampler(dc, cfg_for(max(1, args.warmup)))
    if args.warmup > 0:
        if world > 1:
            D.run_native(sampler, ex)
        else:
            sampler.run()
    sampler.close()
    # A circuit small enough for the specialised soft pass has it compiled by
    # NVRTC in the background on first use (once per process): let that end
    # before timing, as CUDA module loading would.
    from paper_2502_08673_b200 import jit_quiesce
    jit_quiesce()
    sampler = Sampler(dc, cfg_for(args.steps))
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    if world == 1:
        # satgrad::run in C++ (sgx_run): device time from CUDA events on the
        # sampler stream around the whole run.
        with ClockSampler(dev) as clk:
            t0 = time.perf_counter()
            st = sampler.run()
            torch.cuda.synchronize(dev)
            wall = time.perf_counter() - t0
        device_s = st.device_ms / 1000.0
        global_unique = st.unique_count
        restarts_done, attempts, launches, ph = st.restarts + 1, st.attempts, st.launches, st.phase_ms
    else:
        # Sample sharding, the loop in C++ (sgx_run_sharded): one NCCL
        # all-gather of the harvest's new fingerprints per harvest, on the
        # sampler's stream.  Every harvest synchronises the host with its
        # device, so the timed wall clock is device-bound.  Max over ranks.
        with ClockSampler(dev) as clk:
            t0 = time.perf_counter()
            sst = D.run_native(sampler, ex)
            torch.cuda.synchronize(dev)
            wall = time.perf_counter() - t0
        t_dev = torch.tensor([wall], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t_dev, op=dist.ReduceOp.MAX)
        device_s = float(t_dev.item())
        global_unique = sst.unique_count
        # this rank's kernels and device phase times (rank 0 reports)
        restarts_done, attempts = sst.restarts + 1, sst.attempts
        launches, ph = sampler.launch_count(), sampler.phase_times()
    if dist:
        dist.barrier()
    sampler.close()

    # e2e through the public API from host buffers: circuit + CNF upload
    # (H2D), the run, every solution key fetched to host memory (D2H).
    e2e_cfg = cfg_for(args.steps)
    e2e_cfg.solution_capacity = 0  # library defaults, as a user calling run() gets them
    if world == 1:  # warm-up of the public path (host result mapping, pool)
        del run_instance(inst, e2e_cfg, device=dev).solutions.keys
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    e2e_keys = None
    if world == 1:
        res = run_instance(inst, e2e_cfg, device=dev)
        e2e_unique, d2h = res.stats.unique_count, res.solutions.keys.nbytes
        e2e_keys = res.solutions.keys
    else:
        dc2 = DeviceCircuit.from_instance(inst, device=dev)
        s2 = Sampler(dc2, e2e_cfg)
        est = D.run_native(s2, ex)
        e2e_keys = s2.fetch()
        d2h = e2e_keys.nbytes
        e2e_unique = est.unique_count
        s2.close()
        dc2.close()
    e2e_wall = time.perf_counter() - t0
    if dist:
        t_e = torch.tensor([e2e_wall], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t_e, op=dist.ReduceOp.MAX)
        e2e_wall = float(t_e.item())
    h2d = sum(x.nbytes for x in (inst.kind, inst.a, inst.b, inst.var, inst.out_var, inst.out_tgt,
                                 inst.cpi, inst.ucpi, inst.clause_ptr, inst.clause_lit))
    # 0 invalid: every solution the public API returned re-verified on the
    # device against the CNF (and for duplicates), outside the timed region.
    chk = dc.verify_keys(e2e_keys)
    if dist:  # each rank stores the solutions it won: sum over ranks
        t_i = torch.tensor([chk["invalid"], chk["checked"]], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(t_i, op=dist.ReduceOp.SUM)
        chk["invalid"], chk["checked"] = int(t_i[0].item()), int(t_i[1].item())
    del e2e_keys
    if ex is not None:
        ex.close()
    e2e = {"value": e2e_unique / e2e_wall, "unit": UNIT,
           "h2d_bytes_per_step": int(h2d / args.steps), "d2h_bytes_per_step": int(d2h / args.steps),
           "wall_s": e2e_wall}

    if rank != 0:
        return
    value = global_unique / device_s if device_s > 0 else 0.0
    ncone, cpi = info["cone_nodes"], info["cpi"]
    roofline = None
    if ph is not None:
        n_steps = args.steps * args.iterations
        # Dominant kernel roofline (SURVEY.md 8(d) compulsory-tape model).
        kernels = {
            "k_forward": (ph["forward"], n_steps, 4 * (cpi + ncone) * batch),
            "k_backward": (ph["backward"], n_steps, 4 * (ncone + 2 * cpi) * batch),
        }
        dom = max(kernels, key=lambda k: kernels[k][0])
        t_ms, nl, bytes_per_launch = kernels[dom]
        avg_s = (t_ms / max(1, nl)) / 1000.0
        peak, peak_kind = peaks()
        achieved = bytes_per_launch / avg_s / 1e9 if avg_s > 0 else 0.0
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"ncu_{name}.json")
        if os.path.exists(prof):
            with open(prof) as f:
                traffic = json.load(f).get(dom, {}).get("dram_bytes_per_launch")
        roofline = {"kernel": dom, "bound": "hbm", "achieved": achieved, "peak": peak,
                    "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": traffic, "algorithmic_bytes_per_launch": bytes_per_launch,
                    "avg_launch_ms": avg_s * 1000.0}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_reference(name, ref_batch, args.iterations, 1, steps=1)
        cpu = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        if cpu["kind"] == "reference":  # the reference's default precision (sampler.hpp:32), beside f32
            c64 = cpu_reference(name, ref_batch, args.iterations, 1, steps=1, f32=False)
            cpu["f64"] = {"value": c64["value"], "sample": c64["sample"]}
    ttk = None
    if world == 1 and not args.no_ttk:
        ttk = time_to_1k(dev, with_cpu=not args.no_cpu_baseline)

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * device_s / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic",
        "config": {"workload": name, "batch": batch, "global_batch": batch * world,
                   "iterations": args.iterations, "lr": 10.0, "seed": 1,
                   "parallelism": f"sample-shard x{world}",
                   "l2": "inputs > L2 (tape %.1f GB)" % (4 * ncone * batch / 1e9)},
        "unique": global_unique, "restarts": restarts_done, "attempts": attempts,
        "invalid": chk["invalid"], "verified": chk["checked"],
        "wall_s": wall, "device_s": device_s,
        "phase_ms": {k: round(v, 3) for k, v in ph.items()} if ph else None,
        "gpu_launches": launches,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "time_to_1k": ttk,
        "e2e": e2e,
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c4_blasted", choices=sorted(WORKLOADS))
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--iterations", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttk", action="store_true", help="skip the time-to-1k measurement")
    args = ap.parse_args()
    world, rank, local, dist = dist_setup(args)
    try:
        if args.impl == "reference":
            run_reference_arm(args, world, rank)
        else:
            run_b200_arm(args, world, rank, local, dist)
    finally:
        if dist:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
