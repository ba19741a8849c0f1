"""Per-kernel instruction count, occupancy and top stall reasons from an ncu report (raw page CSV)."""
import csv
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
for row in r[2:]:
    d = dict(zip(h, row))
    print(d["Kernel Name"][:40], "us", d["gpu__time_duration.sum"], "inst", d["smsp__inst_executed.sum"], "regs",
          d["launch__registers_per_thread"], "warps%", d["sm__warps_active.avg.pct_of_peak_sustained_active"],
          "dram MB", round((float(d["dram__bytes_read.sum"]) + float(d["dram__bytes_write.sum"])), 2))
    st = []
    for k, v in d.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(v)))
            except ValueError:
                pass
    st.sort(key=lambda x: -x[1])
    print("    stalls/issue:", ", ".join(f"{k} {v:.2f}" for k, v in st[:7]))
