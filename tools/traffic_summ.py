"""Summarise tools/gpu_traffic.sh captures: per kernel, ms and DRAM GB."""
import csv
import glob
import sys
from collections import defaultdict

for f in sorted(glob.glob(sys.argv[1])):
    lines = [l for l in open(f) if l.startswith('"')]
    acc = defaultdict(lambda: defaultdict(list))
    for r in csv.DictReader(lines):
        k = r["Kernel Name"].split("(")[0].replace("void ", "")
        v = float(r["Metric Value"].replace(",", ""))
        u = r["Metric Unit"]
        v *= {"Gbyte": 1, "Mbyte": 1e-3, "Kbyte": 1e-6, "byte": 1e-9, "msecond": 1, "usecond": 1e-3,
              "nsecond": 1e-6}.get(u, 1)
        acc[k][r["Metric Name"]].append(v)
    out = []
    for k, m in acc.items():
        g = lambda n: sum(m[n]) / max(1, len(m[n]))
        out.append(f"{k}: {g('gpu__time_duration.sum'):.3f} ms rd {g('dram__bytes_read.sum'):.2f} "
                   f"wr {g('dram__bytes_write.sum'):.2f} GB L2hit {g('lts__t_sector_hit_rate.pct'):.0f}%")
    print(f.split("/")[-1], "|", " | ".join(out))
