"""Host-only checks of the backward pass split (SGX_BWD_SPLIT, sgx_layout.cpp):
splitting wide levels into several passes keeps every record (same count, same
multiset of records per node run) and only adds passes; the kernels' results
are held bit-exact by the GPU golden tests."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, sys
sys.path.insert(0, %r)
from paper_2502_08673_b200 import load_instance
from paper_2502_08673_b200.sampler import layout_stats
out = {}
for name in ("c2_iscas", "c4_blasted"):
    i = load_instance(name)
    out[name] = layout_stats(i.cnf, i.circuit, i.paths)
print(json.dumps(out))
""" % ROOT


def stats(env_extra):
    env = dict(os.environ, SGX_TRACE="1", SGX_NO_LAYOUT_CACHE="1", **env_extra)
    r = subprocess.run([sys.executable, "-c", PROBE], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    passes = [int(line.split("backward ")[1].split(" passes")[0])
              for line in r.stderr.splitlines() if "staged blocks: backward" in line]
    maxblk = [int(line.split("max ")[1].split(" int4")[0])
              for line in r.stderr.splitlines() if "staged blocks: backward" in line]
    return json.loads(r.stdout.strip().splitlines()[-1]), passes, maxblk


@pytest.mark.parametrize("cap", ["160", "100"])
def test_split_keeps_records_and_adds_passes(cap):
    base, p0, m0 = stats({"SGX_BWD_SPLIT": "0"})
    split, p1, m1 = stats({"SGX_BWD_SPLIT": cap})
    for name in base:
        assert split[name]["bwd_ops"] == base[name]["bwd_ops"], name
        assert split[name]["soft_levels"] == base[name]["soft_levels"], name
    assert len(p0) == len(p1) == 2
    for a, b, ma, mb in zip(p0, p1, m0, m1):
        assert b > a          # wide levels became several passes
        assert mb < ma        # and the largest staged block shrank
    if cap == "160":
        assert max(m1) <= 192  # what lets the third data stage fit at 4 CTAs per SM
