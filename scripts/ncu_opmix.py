"""Executed-instruction mix by SASS opcode of the first kernel in an ncu report:
python scripts/ncu_opmix.py a.ncu-rep [b.ncu-rep ...] (b: all its kernels summed)"""
import collections
import csv
import io
import subprocess
import sys


def mix(rep, first_only):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    c = collections.Counter()
    nk = 0
    hdr = None
    for r in csv.reader(io.StringIO(txt)):
        if r and r[0] == "Kernel Name":
            nk += 1
            if first_only and nk > 1:
                break
            continue
        if r and r[0] == "Address":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            op = r[1].strip().split()
            if not op:
                continue
            o = op[0]
            if o.startswith("@"):
                o = op[1]
            c[o.split(".")[0]] += int(float(r[hdr.index("Instructions Executed")] or 0))
    return c


a = mix(sys.argv[1], True)
b = mix(sys.argv[2], False) if len(sys.argv) > 2 else None
keys = sorted(set(a) | set(b or {}), key=lambda k: -(a.get(k, 0) - (b or {}).get(k, 0)))
print(f"{'op':12s} {'A':>12s} {'B':>12s} {'A-B':>12s}")
for k in keys[:30]:
    print(f"{k:12s} {a.get(k, 0):12d} {(b or {}).get(k, 0):12d} {a.get(k, 0) - (b or {}).get(k, 0):12d}")
print("total", sum(a.values()), sum((b or {}).values()))
