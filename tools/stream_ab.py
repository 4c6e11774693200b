"""Device time of a C2 10-restart run: host streaming on/off x presized/default sizing."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *  # noqa
from paper_2502_08673_b200.sampler import device_context
device_context(0)
inst = load_instance("c2_iscas")
dc = DeviceCircuit.from_instance(inst)
for cap in (0, 60 * 65536):
    for stream in (False, True):
        cfg = SamplerConfig(batch=65536, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=9,
                            solution_capacity=cap)
        ds = []
        for _ in range(3):
            s = Sampler(dc, cfg)
            if stream:
                s.set_host_stream(True)
            ds.append(round(s.run().device_ms, 1))
            if stream:
                del_k = s.take()
                del del_k
            s.close()
        print("capacity", cap, "stream", stream, ds, flush=True)
