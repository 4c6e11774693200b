"""Is the first run of a freshly created sampler slow (bench times exactly that)?"""
import sys
import time
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *  # noqa
from paper_2502_08673_b200.sampler import device_context
device_context(0)
name = sys.argv[1] if len(sys.argv) > 1 else "c3a_or50"
batch = {"c3a_or50": 1 << 20, "c2_iscas": 65536}[name]
inst = load_instance(name)
dc = DeviceCircuit.from_instance(inst)
cfg = SamplerConfig(batch=batch, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=4,
                    solution_capacity=30 * batch)
for rep in range(4):
    t0 = time.perf_counter()
    s = Sampler(dc, cfg)
    t1 = time.perf_counter()
    runs = [round(s.run().device_ms, 1) for _ in range(3)]
    s.close()
    print(name, "fresh sampler: create %.1f ms, runs" % (1000 * (t1 - t0)), runs, flush=True)
