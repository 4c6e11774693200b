import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import load_instance, run_instance, SamplerConfig, RestartPolicy, DeviceCircuit, Sampler
inst = load_instance("c4_blasted")
cfg = SamplerConfig(batch=65536, iterations=5, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=9)
REPS = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for k in range(REPS):
    t = time.perf_counter(); r = run_instance(inst, cfg, device=0); t1 = time.perf_counter()
    print(f"run_instance: device {r.stats.device_ms if hasattr(r.stats,'device_ms') else '?'} ms wall {1e3*(t1-t):.1f} ms unique {r.stats.unique_count}", flush=True)
    del r
if len(sys.argv) > 2 and sys.argv[2] == 'e2e':
    sys.exit(0)
dc = DeviceCircuit.from_instance(inst)
for k in range(3):
    s = Sampler(dc, cfg); t = time.perf_counter(); st = s.run(); t1 = time.perf_counter(); keys = s.fetch(); t2 = time.perf_counter()
    print(f"Sampler.run: device {st.device_ms:.1f} ms run wall {1e3*(t1-t):.1f} fetch {1e3*(t2-t1):.1f} ms unique {st.unique_count}", flush=True)
    s.close(); del keys
