"""Per-instance device time of a few C5 instances as the sweep runs them (design aid)."""
import sys
sys.path.insert(0, '/root/repo')
from paper_2502_08673_b200.sweep import _device_runner, manifest, family, FAMILY_BATCH  # noqa
import torch
torch.cuda.set_device(0)
run_one = _device_runner(0, None)
names = [m["name"] for m in manifest()]
run_one(names[0], 1024, 0, 1)
for n in names[:4] + names[16:18] + names[32:34]:
    u, sec = run_one(n, FAMILY_BATCH[family(n)], 0, 1)
    print(n, u, "%.2f ms" % (sec * 1e3), "%.0f M/s" % (u / sec / 1e6), flush=True)
