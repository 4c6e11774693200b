"""Host timing of the time-to-1k end-to-end path (run() with a quota)."""
import sys
import time
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *  # noqa
from paper_2502_08673_b200.sampler import device_context
device_context(0)
inst = load_instance("c3a_or50")
cfg = SamplerConfig(batch=1 << 20, iterations=5, seed=1, max_solutions=1000, restart=RestartPolicy.REINIT_ON_EXHAUST)
for rep in range(4):
    t = [time.perf_counter()]
    dc = DeviceCircuit.from_instance(inst); t.append(time.perf_counter())
    s = Sampler(dc, cfg); t.append(time.perf_counter())
    s.set_host_stream(True); t.append(time.perf_counter())
    st = s.run(); t.append(time.perf_counter())
    k = s.take(); t.append(time.perf_counter())
    s.close(); t.append(time.perf_counter())
    dc.close(); t.append(time.perf_counter())
    d = [1000 * (b - a) for a, b in zip(t, t[1:])]
    print(rep, "circuit %.2f create %.2f stream %.2f run %.2f (dev %.2f) take %.2f sfree %.2f cfree %.2f" % (*d[:4], st.device_ms, *d[4:]), flush=True)
    t0 = time.perf_counter(); r = run_instance(inst, cfg); print("   run_instance %.2f ms" % (1000 * (time.perf_counter() - t0)))
