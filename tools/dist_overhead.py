"""run_sharded (world 1, NCCL) vs sgx_run on the same sampler: the cost of the
sharded protocol per harvest (collectives, host syncs, no step/harvest overlap)."""
import os
import sys
import time
sys.path.insert(0, '/root/repo')
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29533")
import torch
import torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
from paper_2502_08673_b200 import *  # noqa
from paper_2502_08673_b200.dist import DeviceShard, TorchExchange, run_sharded
name = sys.argv[1] if len(sys.argv) > 1 else "c2_iscas"
batch = {"c3a_or50": 1 << 20, "c2_iscas": 65536}[name]
inst = load_instance(name)
dc = DeviceCircuit.from_instance(inst)
cfg = SamplerConfig(batch=batch, seed=1, restart=RestartPolicy.REINIT_ON_EXHAUST, max_restarts=4,
                    solution_capacity=40 * batch)
s = Sampler(dc, cfg)
s.run()
for _ in range(2):
    st = s.run()
    print(name, "sgx_run device %.1f ms unique %d" % (st.device_ms, st.unique_count), flush=True)
sh = DeviceShard(s)
ex = TorchExchange(device="cuda:0")
for _ in range(3):
    s.L.sgx_run  # noqa
    from paper_2502_08673_b200 import _lib
    _lib.check(s.L.sgx_set_host_stream(s.h, 0))
    s.run()  # reset the solution set (sgx_run resets it)
    torch.cuda.synchronize()
    # restart from an empty table: a fresh sampler keeps the comparison fair
    s2 = Sampler(dc, cfg)
    sh2 = DeviceShard(s2)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = run_sharded(sh2, ex, cfg, 0, 1, sh2.stride)
    torch.cuda.synchronize()
    print(name, "run_sharded wall %.1f ms unique %d" % (1000 * (time.perf_counter() - t0), r.unique_count), flush=True)
    s2.close()
dist.destroy_process_group()
