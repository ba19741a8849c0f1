"""DRAM bytes (read + write) per launch of each GP kernel from one `ncu --set full` capture, merged into
profiles/traffic.json under the configuration key "<cells>x<grid>" that bench.py reads into
roofline.traffic.  Usage: ncu_traffic.py REPORT OUT_JSON [KEY]"""
import csv
import json
import subprocess
import sys

MAP = {"k_density_scatter_win": "density_scatter", "k_density_scatter_limbs": "density_scatter", "k_dens_grad": "dens_grad", "k_cells": "cells",
       "k_density_bins": "density_bins", "k_finalize": "finalize", "k_wa_": "wirelength_pp"}
raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
per = {}
for row in r[2:]:
    d = dict(zip(h, row))
    name = d["Kernel Name"]
    key = next((v for k, v in MAP.items() if k in name), None)
    if key is None:
        continue
    b = float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])
    unit = h and r[1][h.index("dram__bytes_read.sum")]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    per.setdefault(key, {}).setdefault(name, []).append(b * scale)
out = {}
for key, kernels in per.items():  # sum over the kernels of one stage, mean over repeated launches
    out[key] = round(sum(sum(v) / len(v) for v in kernels.values()))
out["_source"] = sys.argv[1].split("/")[-1] + " (ncu --set full --clock-control none, one GP iteration)"
key = sys.argv[3] if len(sys.argv) > 3 else "1100000x1024"
try:
    allk = json.load(open(sys.argv[2]))
except (OSError, ValueError):
    allk = {}
allk[key] = out
json.dump(allk, open(sys.argv[2], "w"), indent=1)
print(key, out)
