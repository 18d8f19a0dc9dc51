"""Per CUDA source line: warp instructions executed and stall samples, from
an ncu report captured with -lineinfo (python tools/ncu_lines.py rep [top])."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows, cur, hdr = [], None, None
for rec in csv.reader(out):
    if not rec:
        continue
    if rec[0] == "File Path":
        cur = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("Function Name",):
        continue
    try:
        ln = int(rec[0])
    except ValueError:
        continue
    if rec[2] != "-":  # sass rows under a source line carry an address; keep source-line totals
        continue
    d = dict(zip(hdr[4:], rec[4:]))
    rows.append((cur, ln, rec[1].strip()[:70], int(d.get("Instructions Executed", 0) or 0),
                 int(d.get("# Samples", 0) or 0)))
tot_i = sum(r[3] for r in rows)
tot_s = sum(r[4] for r in rows)
print(f"total warp instructions {tot_i}, samples {tot_s}")
for r in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{r[0]:12s}:{r[1]:<5d} {100*r[3]/max(tot_i,1):5.1f}% instr {100*r[4]/max(tot_s,1):5.1f}% smp  {r[2]}")
