"""A/B of the soft-pass kernels: HBM tape vs the circuit-specialised (JIT) one.

    python tools/jit_ab.py [workload ...]

Per workload at its bench batch: run() device time, per-phase times, unique/s,
and the soft step time per iteration, for SoftKernel.HBM and SoftKernel.JIT
(same seed: the runs must agree exactly).
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402

from paper_2502_08673_b200 import DeviceCircuit, Sampler, SamplerConfig, SoftKernel, load_instance  # noqa: E402

BATCH = {"c3a_or50": 1 << 20, "c3b_or100": 1 << 20, "c1b_random": 1 << 20, "c1a_planted3sat": 1 << 18,
         "mux_chain14": 1 << 20}


def one(name, mode, reps=3):
    i = load_instance(name)
    dc = DeviceCircuit.from_instance(i)
    cfg = SamplerConfig(batch=BATCH.get(name, 65536), iterations=5, seed=1, soft_kernel=mode)
    s = Sampler(dc, cfg)
    s.run()  # warm
    best = None
    for _ in range(reps):
        st = s.run()
        if best is None or st.device_ms < best.device_ms:
            best = st
    keys = s.fetch()
    info = s.soft_info()
    s.close()
    dc.close()
    return best, keys, info


def main(names):
    for name in names:
        res = {}
        for mode in (SoftKernel.HBM, SoftKernel.JIT):
            st, keys, info = one(name, mode)
            res[mode] = (st, keys)
            ph = st.phase_ms
            n_steps = len(st.loss_trace)
            print(f"{name:16s} {mode.name:4s} device {st.device_ms:8.3f} ms  unique {st.unique_count:9d} "
                  f"({st.unique_count / st.device_ms * 1e3 / 1e6:8.2f} M/s)  step/iter "
                  f"{ph['step'] / max(1, n_steps):7.4f} ms  fwd {ph['forward']:.3f} bwd {ph['backward']:.3f} "
                  f"harvest {ph['harvest']:.3f}  [{info['last']}, compile {info['jit_compile_ms']:.0f} ms]",
                  flush=True)
        a, b = res[SoftKernel.HBM], res[SoftKernel.JIT]
        same = a[0].new_unique == b[0].new_unique and np.array_equal(a[1], b[1])
        print(f"{name:16s} identical runs: {same}", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c3a_or50", "c3b_or100", "c1b_random"])
