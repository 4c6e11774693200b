import sys; sys.path.insert(0, '/root/repo')
import numpy as np
from paper_2502_08673_b200 import *
from oracle.oracle import PortLib
name, batch = sys.argv[1], int(sys.argv[2])
i = load_instance(name); P = PortLib()
s = Sampler(DeviceCircuit.from_instance(i), SamplerConfig(batch=batch, seed=3, iterations=3))
s.init(1)
v0 = P.init_soft_inputs(batch, len(i.cpi), 3, 1).astype(np.float32)
s.step()
tape, _ = P.forward(i, i.cpi, P.embed(v0))
dv, dp = P.backward(i, i.cpi, tape, v0)
v1 = (v0 - np.float32(10.0) * dv).astype(np.float32)
got = s.logits()
rows, cols = np.nonzero(got.view(np.uint32) != v1.view(np.uint32))
print('n bad', len(rows), 'rows', sorted(set(rows.tolist()))[:20])
for r, c in list(zip(rows, cols))[:6]:
    ddv = (v0[r, c] - got[r, c]) / 10
    print(r, c, 'v0', v0[r, c], 'want', v1[r, c], 'got', got[r, c], 'dv', dv[r, c], 'dev dv~', ddv, 'dp', dp[r,c])
    print('   row tape', tape[:, r])
