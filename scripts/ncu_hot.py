"""Hottest SASS lines of an ncu report (warp-stall samples): python scripts/ncu_hot.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = rows[1]
si, src, ex = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
body = []
for r in rows[2:]:                      # the first kernel's section only
    if r and r[0] == "Kernel Name":
        break
    if len(r) > si:
        body.append(r)
tot = sum(float(r[si] or 0) for r in body)
print(f"total samples {tot:.0f}, instructions {sum(float(r[ex] or 0) for r in body):.0f}")
for i, r in sorted(enumerate(body), key=lambda t: -float(t[1][si] or 0))[:n]:
    print(f"{i:5d} {float(r[si]):7.0f} {100 * float(r[si]) / tot:5.1f}% exec {r[ex]:>9}  {r[src].strip()[:80]}")
