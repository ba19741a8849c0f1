"""Aggregate an ncu --metrics gpu__time_duration.sum CSV by kernel name: launches, total us, share."""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
agg, tot = collections.OrderedDict(), 0.0
for r in rows:
    name = r[4].split("(")[0].replace("tdpg::", "").replace("void ", "")[:56]
    v, unit = float(r[14]), r[13]
    us = {"nsecond": v / 1e3, "ns": v / 1e3, "usecond": v, "us": v, "msecond": v * 1e3, "ms": v * 1e3}.get(unit, v / 1e3)
    a = agg.setdefault(name, [0, 0.0])
    a[0] += 1
    a[1] += us
    tot += us
print(f"launches {len(rows)}, total {tot:.1f} us")
for k, (n, us) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"  {k:58s} x{n:3d} {us:9.1f} us {100 * us / tot:5.1f}%")
