"""Drive one workload's soft steps for an ncu capture of the specialised kernel.

    python tools/prof_jit.py [workload] [batch] [steps] [hbm|jit]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2502_08673_b200 import DeviceCircuit, Sampler, SamplerConfig, SoftKernel, load_instance  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3a_or50"
batch = int(sys.argv[2]) if len(sys.argv) > 2 else 1 << 20
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
mode = SoftKernel.HBM if (len(sys.argv) > 4 and sys.argv[4] == "hbm") else SoftKernel.JIT
s = Sampler(DeviceCircuit.from_instance(load_instance(name)),
            SamplerConfig(batch=batch, iterations=steps, seed=1, soft_kernel=mode))
s.init(0)
for _ in range(steps):
    s.step()
print(name, batch, s.soft_info())
s.close()
