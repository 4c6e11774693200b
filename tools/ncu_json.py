"""profiles/ncu_<workload>.json from an `ncu --set full` report: per dominant
kernel family, the DRAM bytes of one launch (bench.py roofline `traffic`).

usage: python tools/ncu_json.py REPORT.ncu-rep WORKLOAD "SOURCE NOTE"
"""
import csv
import json
import subprocess
import sys

rep, name, note = sys.argv[1], sys.argv[2], sys.argv[3]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]


def val(r, key):
    i = hdr.index(key)
    x = float(r[i].replace(",", ""))
    u = units[i]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "msecond": 1, "usecond": 1e-3,
             "nsecond": 1e-6}.get(u, 1)
    return x * scale


fam = {"k_backward": "k_backward", "k_forward": "k_forward", "k_harvest_smem": "k_harvest",
       "k_harvest_live": "k_harvest", "k_harvest_lw": "k_harvest", "k_keys_spill": "k_keys"}
res = {}
for r in rows[2:]:
    kname = r[hdr.index("Kernel Name")]
    for key, tag in fam.items():
        if key in kname and tag not in res:
            rd, wr = val(r, "dram__bytes_read.sum"), val(r, "dram__bytes_write.sum")
            res[tag] = {"kernel": kname.split("(")[0], "dram_bytes_per_launch": rd + wr,
                        "dram_read_bytes": rd, "dram_write_bytes": wr,
                        "duration_ms_ncu": val(r, "gpu__time_duration.sum"),
                        "dram_pct_of_peak": float(r[hdr.index(
                            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")]),
                        "warps_active_pct": float(r[hdr.index(
                            "sm__warps_active.avg.pct_of_peak_sustained_active")]),
                        "source": note}
json.dump(res, open(f"profiles/ncu_{name}.json", "w"), indent=1)
print(json.dumps(res, indent=1))
