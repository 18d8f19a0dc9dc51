"""Summarise an ncu report: headline metrics and the SASS lines with the most
stall samples (python tools/ncu_hot.py report.ncu-rep [top])."""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(det.splitlines()))
h = r[0]
want = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Executed Ipc Active", "Achieved Active Warps Per SM", "Registers Per Thread",
        "Executed Instructions", "Issued Instructions")
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Metric Name']:32s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(src.splitlines()))
h = r[1]
rows = r[2:]
iS, iE = h.index("# Samples"), h.index("Instructions Executed")
stalls = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
tot = sum(int(x[iS]) for x in rows)
print("samples", tot, "warp instructions", sum(int(x[iE]) for x in rows))
agg = Counter()
for x in rows:
    for k in stalls:
        agg[k] += int(x[h.index(k)])
print("stalls:", ", ".join(f"{k[6:]} {100*v/max(tot,1):.1f}%" for k, v in agg.most_common(8)))
for i, x in enumerate(rows):
    x.append(i)
for x in sorted(sorted(rows, key=lambda x: -int(x[iS]))[:top], key=lambda x: x[-1]):
    st = max(((int(x[h.index(k)]), k) for k in stalls))
    print(f"{x[-1]:5d} {x[1][:56]:56s} {x[iS]:>6s} {x[iE]:>9s} {st[1][6:]}")
