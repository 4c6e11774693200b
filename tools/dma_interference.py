"""Does a D2H stream beside the soft passes slow them (and why)?  Sampler.run()
on C4 (device-timed, no host streaming) while a side thread copies 220 MB
chunks (one harvest's new keys) every 10 ms: device -> pinned host
(cudaHostAlloc), device -> device, or nothing.  Design aid (DESIGN.md e2e)."""
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08673_b200 import DeviceCircuit, RestartPolicy, Sampler, SamplerConfig, load_instance  # noqa: E402

inst = load_instance("c4_blasted")
cfg = SamplerConfig(batch=65536, iterations=5, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=9)
dc = DeviceCircuit.from_instance(inst)
n = 220 << 20
src = torch.empty(n, dtype=torch.uint8, device="cuda:0")
dst_h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
dst_d = torch.empty(n, dtype=torch.uint8, device="cuda:0")
side = torch.cuda.Stream()


def run(mode, chunk=n, gap=0.010):
    stop = threading.Event()
    count = [0]

    def loop():
        with torch.cuda.stream(side):
            while not stop.is_set():
                if mode == "h2d_none":
                    break
                (dst_h if mode == "d2h" else dst_d)[:chunk].copy_(src[:chunk], non_blocking=True)
                side.synchronize()
                count[0] += chunk / n
                time.sleep(gap)

    th = threading.Thread(target=loop)
    s = Sampler(dc, cfg)
    th.start()
    st = s.run()
    stop.set()
    th.join()
    s.close()
    return st.device_ms, count[0]


for rep in range(2):
    for mode, chunk, gap in (("h2d_none", n, 0.01), ("d2h", n, 0.01), ("d2d", n, 0.01), ("d2h", 32 << 20, 0.0015),
                             ("d2h", 4 << 20, 0.0002)):
        ms, c = run(mode, chunk, gap)
        print(f"{mode:9s} chunk {chunk >> 20:4d} MB gap {gap * 1e3:4.1f} ms: device {ms:7.1f} ms  "
              f"side copies {c:.1f} x 220 MB", flush=True)
