"""Per-kernel device time per GP iteration from an ncu launch list (last 3 iterations)."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hi], rows[hi + 1:]
iK, iM, iV, iID = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
per = {}
for r in data:
    name = r[iK].split("(")[0].replace("void ", "")
    per.setdefault(r[iID], {})["name"] = name
    per[r[iID]][r[iM]] = float(r[iV].replace(",", ""))
ids = sorted(per, key=int)
cells = [k for k, i in enumerate(ids) if per[i]["name"].endswith("k_cells")]
start, end = cells[-4] + 1, cells[-1]
agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
for i in ids[start:end + 1]:
    p = per[i]
    a = agg[p["name"][:40]]
    a[0] += 1
    a[1] += p.get("gpu__time_duration.sum", 0)
    a[2] += p.get("dram__bytes_read.sum", 0)
    a[3] += p.get("dram__bytes_write.sum", 0)
tot = sum(v[1] for v in agg.values()) / 3
print(f"launches {len(ids)}; per iteration: {tot / 1000:.1f} us over {sum(v[0] for v in agg.values()) // 3} kernels")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"  {k:40s} x{v[0] // 3:2d} {v[1] / 3 / 1000:8.2f} us  rd {v[2] / 3 / 1e6:7.1f} MB  wr {v[3] / 3 / 1e6:6.1f} MB")
