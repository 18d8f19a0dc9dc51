"""Sum an ncu launch list (--metrics gpu__time_duration.sum --csv) by kernel:
python tools/ncu_sum.py launches.csv [substring ...] prints the total kernel
time, then count / total / mean per kernel whose name holds a substring (all
kernels when none is given)."""
import csv
import re
import sys
from collections import defaultdict

path, keys = sys.argv[1], sys.argv[2:]
lines = open(path, errors="replace").read().splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
rows = list(csv.DictReader(lines[start:]))
per = defaultdict(list)
for r in rows:
    if r.get("Metric Name") != "gpu__time_duration.sum":
        continue
    v = float(r["Metric Value"].replace(",", ""))
    unit = r.get("Metric Unit", "ns")
    us = v / 1e3 if unit == "ns" else v * 1e3 if unit == "msecond" else v
    name = r["Kernel Name"].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    name = re.sub(r"\(.*", "", name)
    name = name.split("<")[0] if "cub" not in name else name[:60]
    per[name].append(us)
tot = sum(sum(v) for v in per.values())
print(f"{path}: {sum(len(v) for v in per.values())} launches, {tot / 1e3:.3f} ms")
for name, v in sorted(per.items(), key=lambda x: -sum(x[1])):
    if keys and not any(k in name for k in keys):
        continue
    print(f"  {name:60s} {len(v):5d}x {sum(v) / 1e3:8.3f} ms  mean {sum(v) / len(v):8.1f} us")
