import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from test_gpu_dist import run_two_shards
from paper_2502_08673_b200 import *
from oracle.oracle import PortLib
inst = load_instance('c1b_random')
cfg = SamplerConfig(batch=700, iterations=2, seed=2, max_solutions=100000, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=3)
big = SamplerConfig(**{**cfg.__dict__, "batch": 1400})
want = run_instance(inst, big)
print('single', want.stats.unique_count, want.stats.new_unique, want.stats.restarts)
p = PortLib().run(inst, batch=1400, iterations=2, seed=2, max_solutions=100000, restart=True)
print('port  ', p.unique, p.new_unique, p.restarts)
for t in range(3):
    stats, keys = run_two_shards(inst, cfg)
    print('shards', stats[0].unique_count, stats[0].new_unique, stats[0].restarts, [len(k) for k in keys])
