"""Small sampler runs for compute-sanitizer (memcheck / racecheck)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *  # noqa
from paper_2502_08673_b200.sampler import device_context
device_context(0)
for name, b in (("c1b_random", 1024), ("c3a_or50", 4096), ("c2_iscas", 2048)):
    inst = load_instance(name)
    res = run_instance(inst, SamplerConfig(batch=b, iterations=2, seed=1))
    print(name, res.stats.unique_count, flush=True)
