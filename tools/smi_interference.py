"""Does nvidia-smi polling (the bench's clock sampler) stall a sync-heavy run?"""
import subprocess
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
s = Sampler(dc, cfg)
s.run()
for mode in ("quiet", "smi", "quiet", "smi-q", "quiet"):
    p = None
    if mode == "smi":
        p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks_event_reasons.active",
                              "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    if mode == "smi-q":
        p = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm", "--format=csv,noheader,nounits",
                              "-lms", "200"], stdout=subprocess.DEVNULL)
        time.sleep(0.5)
    ds = []
    for _ in range(3):
        st = s.run()
        ds.append(round(st.device_ms, 1))
    if p:
        p.terminate()
        p.wait()
    print(name, mode, ds, flush=True)
