"""Where the end-to-end time of run() goes (upload / create / run / fetch / free)."""
import sys, time
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *
from paper_2502_08673_b200.sampler import device_context
import torch
device_context(0)
for name, cfg in [("c3a_or50", SamplerConfig(batch=1 << 20, seed=1, max_solutions=1000, restart=RestartPolicy.REINIT_ON_EXHAUST)),
                  ("c2_iscas", SamplerConfig(batch=65536, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=4))]:
    inst = load_instance(name)
    for rep in range(3):
        t = [time.perf_counter()]
        dc = DeviceCircuit.from_instance(inst); t.append(time.perf_counter())
        s = Sampler(dc, cfg); s.set_host_stream(True); t.append(time.perf_counter())
        st = s.run(); t.append(time.perf_counter())
        k = s.take(); t.append(time.perf_counter())
        s.close(); dc.close(); t.append(time.perf_counter())
        d = [1000 * (b - a) for a, b in zip(t, t[1:])]
        print(name, rep, "upload %.1f create %.1f run %.1f (device %.1f) fetch %.1f free %.1f ms; unique %d" % (*d[:3], st.device_ms, d[3], d[4], st.unique_count))
