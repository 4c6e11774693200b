import sys; sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200 import *
from oracle.oracle import PortLib
inst = load_instance(sys.argv[1] if len(sys.argv) > 1 else 'c1b_random')
for b in (1400, 3000):
    want = PortLib().run(inst, batch=b, iterations=3, seed=2)
    for t in range(2):
        got = run_instance(inst, SamplerConfig(batch=b, iterations=3, seed=2))
        print(b, got.stats.new_unique == want.new_unique, got.stats.new_unique, want.new_unique)
