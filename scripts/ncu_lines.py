"""Per-source-line instruction counts and stall samples of an ncu report
(`--page source --print-source cuda,sass`): python scripts/ncu_lines.py REP [N]."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
hdr = None
fname = ""
for r in csv.reader(out.splitlines()):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[2] == "-":
        try:
            rows.append((int(r[hdr.index("Instructions Executed")]), int(r[hdr.index("Warp Stall Sampling (All Samples)")]),
                         fname, r[0], r[1].strip()[:90]))
        except ValueError:
            pass
tot_i = sum(x[0] for x in rows) or 1
tot_s = sum(x[1] for x in rows) or 1
print(f"total warp instructions {tot_i}, stall samples {tot_s}")
for i, s, f, ln, src in sorted(rows, reverse=True)[:n]:
    print(f"{100 * i / tot_i:5.1f}% inst {100 * s / tot_s:5.1f}% samp  {f}:{ln:5s} {src}")
