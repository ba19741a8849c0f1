"""Top SASS instructions by warp-stall samples for one kernel of an ncu report (source page, SASS view).
usage: python tools/ncu_src_top.py report.ncu-rep kernel_regex [n] [which_launch]"""
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 40
which = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", "regex:" + kre],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
lo = starts[which]
hi = starts[which + 1] if which + 1 < len(starts) else len(rows)
blk = rows[lo:hi]
print(blk[0][1])
hdr_i = [i for i, r in enumerate(blk) if r and r[0] == "Address"][0]
h, data = blk[hdr_i], blk[hdr_i + 1:]
si, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
val = lambda r, k: int(r[k]) if len(r) > k and r[k].isdigit() else 0
tot = sum(val(r, si) for r in data)
print("total stall samples", tot, "instructions", len(data))
for k in sorted(range(len(data)), key=lambda k: -val(data[k], si))[:n]:
    r = data[k]
    print(f"{k:5d} {val(r, si):6d} {100.0 * val(r, si) / max(tot, 1):5.1f}% exec {val(r, ii):9d}  {r[1].strip()[:80]}")
