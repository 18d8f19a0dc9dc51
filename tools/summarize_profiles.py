"""Summaries of ncu outputs for profiles/ (launch list CSV, --set full report).

    python tools/summarize_profiles.py launches gpurun_out/X.csv "<command>" > profiles/Y.md
    python tools/summarize_profiles.py full gpurun_out/X.ncu-rep "<command>" > profiles/Z.md
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path, cmd):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hdr + 1:]:
        if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("void ", "")
        if name.startswith("po::"):
            name = name.replace("po::", "").replace("<unnamed>::", "")
        name = name[:60]
        v = float(r[vi].replace(",", ""))
        unit = h[vi]
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    print("# Kernel launch list (ncu gpu__time_duration, --clock-control none)\n")
    print(f"Command: `{cmd}`\n")
    print("Per-launch times are cold-cache and serialised: compare SHARES, not absolutes.\n")
    print(f"Total kernel time: {tot/1e6:.3f} ms\n")
    print("| kernel | launches | total us | share |\n|---|---:|---:|---:|")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"| {k} | {c} | {v/1e3:.1f} | {100*v/tot:.1f}% |")


def full(path, cmd):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]
    print("# ncu --set full summary\n")
    print(f"Command: `{cmd}`\n")
    ki = h.index("Kernel Name")
    for r in rows[2:]:
        print(f"## {r[ki].split('(')[0]}")
        for w in want:
            if w in h:
                i = h.index(w)
                print(f"- {w}: {r[i]} {units[i]}")
        stalls = []
        for i, k in enumerate(h):
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                try:
                    stalls.append((float(r[i].replace(",", "")), k[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        stalls.sort(reverse=True)
        print("- top stall reasons (samples): " + ", ".join(f"{n} {int(v)}" for v, n in stalls[:4]))


if __name__ == "__main__":
    {"launches": launches, "full": full}[sys.argv[1]](sys.argv[2], sys.argv[3])
