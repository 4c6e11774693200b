"""Print value / phase_ms of every gpurun_out/bench_*.txt (A/B summaries)."""
import glob
import json
import sys

for f in sorted(glob.glob(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/bench_*.txt")):
    lines = [x for x in open(f) if x.startswith("{")]
    if not lines:
        print(f, "no JSON line")
        continue
    d = json.loads(lines[-1])
    ph = d.get("phase_ms", {})
    print(f, round(d.get("value", 0)), {k: ph[k] for k in ("forward", "backward", "harvest") if k in ph},
          d.get("roofline", {}).get("frac"))
