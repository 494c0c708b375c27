"""Fold `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
output of tools/bw_kernels.py into the CUDA-event JSON (last launch per kernel).

usage: python tools/bw_ncu_summary.py bw.json bw_ncu.csv out.json
"""
import csv
import json
import sys
from collections import defaultdict

events, ncu_csv, out = sys.argv[1:4]
rows = list(csv.reader(open(ncu_csv)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h, data = rows[hi], rows[hi + 1:]
kn, mn, mv, mu, idc = (h.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value",
                                            "Metric Unit", "ID"))
scale = {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9,
         "s": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
launch = defaultdict(dict)
for r in data:
    launch[r[idc]][r[mn]] = float(r[mv].replace(",", "")) * scale[r[mu]]
    launch[r[idc]]["name"] = r[kn].split("(")[0].split("::")[-1]
last = {}
for _, d in sorted(launch.items(), key=lambda x: int(x[0])):
    if d["name"].endswith(">") and "kernel" in d["name"] and "distribution" not in d["name"]:
        last[d["name"]] = d
res = json.load(open(events))
peak = res["hbm_peak_gbs"]
kern = []
for name, d in last.items():
    t = d["gpu__time_duration.sum"]
    b = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    kern.append({"kernel": name, "ncu_us": round(t * 1e6, 1), "dram_MB": round(b / 1e6, 1),
                 "dram_GBs": round(b / t / 1e9), "frac_hbm": round(b / t / 1e9 / peak, 3)})
res["ncu_dram"] = {"command": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                              "dram__bytes_write.sum --clock-control none python "
                              "tools/bw_kernels.py --reps 1 (last launch of each kernel)",
                   "kernels": kern}
json.dump(res, open(out, "w"), indent=1)
for k in kern:
    print(f"{k['kernel']:40s} {k['ncu_us']:9.1f} us {k['dram_MB']:9.1f} MB {k['dram_GBs']:6d} GB/s")
