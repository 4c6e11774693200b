"""Small runs of the round-2 kernels for compute-sanitizer (memcheck / racecheck /
synccheck): the warp-synchronous harvest with its TMA record ring
(k_harvest_lw) and the spill key kernel (k_keys_spill), forced on every
instance; the NVRTC soft pass (SoftKernel.JIT); the Adam epilogue; and the
sharded run through the in-process exchange (2 ranks, threads)."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["SGX_HARVEST"] = "lw"
from paper_2502_08673_b200 import (DeviceCircuit, Optimizer, Sampler, SamplerConfig, SoftKernel,  # noqa: E402
                                   load_instance, run_instance)
from paper_2502_08673_b200 import dist as D  # noqa: E402

for name, b in (("c1b_random", 1024), ("c3a_or50", 4096), ("c2_iscas", 2048), ("c4_blasted", 256)):
    inst = load_instance(name)
    res = run_instance(inst, SamplerConfig(batch=b, iterations=2, seed=1))
    print(name, "lw", res.stats.unique_count, flush=True)
inst = load_instance("c3a_or50")
res = run_instance(inst, SamplerConfig(batch=4096, iterations=2, seed=1, soft_kernel=SoftKernel.JIT))
print("c3a_or50 jit", res.stats.unique_count, flush=True)
res = run_instance(inst, SamplerConfig(batch=4096, iterations=2, seed=1, optimizer=Optimizer.ADAM, learning_rate=0.1))
print("c3a_or50 adam", res.stats.unique_count, flush=True)
inst = load_instance("c2_iscas")
ex = D.LocalExchanges(2)
samplers = [Sampler(DeviceCircuit.from_instance(inst), SamplerConfig(batch=1024, row_offset=r * 1024, iterations=2,
                                                                      seed=1)) for r in range(2)]
out = [None, None]
th = [threading.Thread(target=lambda r=r: out.__setitem__(r, D.run_native(samplers[r], ex[r]))) for r in range(2)]
for t in th:
    t.start()
for t in th:
    t.join()
print("c2_iscas sharded x2", [o.unique_count for o in out], flush=True)
for s in samplers:
    s.close()
ex.close()
