"""Many run_instance calls in one process: catch host-side outliers (design aid)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *  # noqa
from paper_2502_08673_b200.sampler import device_context
device_context(0)
inst = load_instance("c2_iscas")
cfg = SamplerConfig(batch=65536, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=9)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 12):
    r = run_instance(inst, cfg)
    del r
