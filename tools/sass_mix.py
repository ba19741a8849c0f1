"""Instruction mix + stall samples per opcode from an ncu report's source (SASS) page.
Usage: python tools/sass_mix.py REPORT.ncu-rep SUBSTRING [top]"""
import collections
import csv
import subprocess
import sys

rep, sub = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 16
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
secs, cur = [], None
for r in csv.reader(raw.splitlines()):
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        secs.append(cur)
    elif cur is not None and r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None:
        cur["rows"].append(r)
seen = set()
for s in secs:
    if sub not in s["name"] or s["name"] in seen:
        continue
    seen.add(s["name"])
    h = s["hdr"]
    ie, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ops, stall, tot, tots = collections.Counter(), collections.Counter(), 0, 0
    for r in s["rows"]:
        if len(r) <= ie or not r[1].strip():
            continue
        w = r[1].strip().split()
        op = (w[1] if w[0].startswith("@") and len(w) > 1 else w[0]).split(".")[0]
        n, sm = int(r[ie] or 0), int(r[st] or 0)
        ops[op] += n
        stall[op] += sm
        tot += n
        tots += sm
    print(s["name"][:90], "warp-inst", tot, "stall samples", tots)
    for k, v in ops.most_common(top):
        print(f"   {k:10s} {v:10d} {100 * v / tot:5.1f}%   stall samples {100 * stall[k] / max(tots, 1):5.1f}%")
