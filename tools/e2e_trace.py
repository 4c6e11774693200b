"""Fine-grained host timing of run() pieces (design aid)."""
import gc
import sys
import time
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *  # noqa
from paper_2502_08673_b200.sampler import device_context
device_context(0)
inst = load_instance("c2_iscas")
cfg = SamplerConfig(batch=65536, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=9)
for rep in range(4):
    t = [time.perf_counter()]
    dc = DeviceCircuit.from_instance(inst); t.append(time.perf_counter())
    s = Sampler(dc, cfg); s.set_host_stream(True); t.append(time.perf_counter())
    st = s.run(); t.append(time.perf_counter())
    k = s.take(); t.append(time.perf_counter())
    s.close(); t.append(time.perf_counter())
    dc.close(); t.append(time.perf_counter())
    del k; gc.collect(); t.append(time.perf_counter())
    d = [1000 * (b - a) for a, b in zip(t, t[1:])]
    print(rep, "circuit %.1f create %.1f run %.1f (dev %.1f) take %.1f sfree %.1f cfree %.1f keysfree %.1f" % (*d[:3], st.device_ms, *d[3:]), flush=True)
    t0 = time.perf_counter(); r = run_instance(inst, cfg); w = time.perf_counter() - t0
    print("   run_instance %.1f ms -> %.2fM solutions/s e2e" % (1000 * w, r.stats.unique_count / w / 1e6), flush=True)
