"""Write profiles/ncu_summary.json (bench.py's roofline.traffic) from the
--set full captures of scripts/gpu_profiles3*.sh, and a text summary of each
capture next to it.  python scripts/update_ncu_summary.py CAPTURE_DIR OUT_DIR"""
import csv
import json
import os
import subprocess
import sys

src, dst = sys.argv[1], sys.argv[2]
os.makedirs(dst, exist_ok=True)


def metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]

    def get(name):
        x = float(v[h.index(name)].replace(",", ""))
        unit = u[h.index(name)]
        return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "msecond": 1e-3,
                    "nsecond": 1e-9, "us": 1e-6, "ms": 1e-3, "ns": 1e-9}.get(unit, 1)
    return (v[h.index("Kernel Name")], get("dram__bytes_read.sum"), get("dram__bytes_write.sum"),
            get("gpu__time_duration.sum"))


MB = {"1": 512 * 512, "2": 4096 ** 2, "3": 16384 ** 2, "4": 8192 ** 2, "4b": 8193 ** 2}
# key -> (captures summed, algorithmic bytes per launch, what)
ENTRIES = {
    "1": (["c1"], 8 * MB["1"], "level 1, 512x512"),
    "2": (["c2"], 8 * MB["2"], "level 1, 4096x4096"),
    "3": (["c3"], 8 * MB["3"], "level 1, 16384x16384"),
    "4": (["c4"], 8 * MB["4"], "level 1, 8192x8192"),
    "4b": (["c4b"], 8 * MB["4b"], "level 1, 8193x8193 (row-grouped TMA, G = 4)"),
    "5": (["c5", "c5_group2"], 8 * (256 * 2048 * 2048 + 32 * 4095 * 3001),
          "level 1 of both groups: 256 x 2048^2 (3-D TMA) + 32 x 4095x3001 (row-grouped TMA, G = 4)"),
    "3_inverse": (["c3_inverse"], 8 * MB["3"], "inverse ring kernel, level 1, 16384x16384"),
    "4_inverse": (["c4_inverse"], 8 * MB["4"], "inverse ring kernel, level 1, 8192x8192"),
    "3_cdf97": (["c3_cdf97"], 8 * MB["3"], "CDF 9/7 level kernel, level 1, 16384x16384"),
    "3_cdf97_inverse": (["c3_cdf97_inverse"], 8 * MB["3"], "CDF 9/7 inverse kernel, level 1, 16384x16384"),
}
out = {"note": ("dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant (level-1) kernel, from "
                "ncu --set full captures of bench.py's own launches (scripts/gpu_profiles3*.sh; cold caches, "
                "serialised, clocks uncontrolled); configs with two level-1 launches (config 5) sum both. "
                "bench.py reports it as roofline.traffic."), "configs": {}}
for key, (caps, alg, what) in ENTRIES.items():
    rd = wr = t = 0.0
    names = []
    for c in caps:
        rep = os.path.join(src, c + ".ncu-rep")
        if not os.path.exists(rep):
            break
        name, r, w, d = metrics(rep)
        rd += r
        wr += w
        t += d
        names.append(name)
        with open(os.path.join(dst, c + "_summary.txt"), "w") as f:
            f.write(subprocess.run([sys.executable, os.path.join(os.path.dirname(__file__), "ncu_summary.py"), rep],
                                   capture_output=True, text=True).stdout)
    else:
        out["configs"][key] = {"kernel": " + ".join(sorted(set(n.split("(")[0].replace("void ", "") for n in names))),
                               "what": what, "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
                               "dram_bytes_per_launch": int(rd + wr), "algorithmic_bytes_per_launch": alg,
                               "traffic_over_algorithmic": round((rd + wr) / alg, 4),
                               "ncu_duration_us": round(t * 1e6, 1),
                               "source": ", ".join(f"profiles/round1/session3/{c}_summary.txt" for c in caps)}
with open(os.path.join(os.path.dirname(__file__), "..", "profiles", "ncu_summary.json"), "w") as f:
    json.dump(out, f, indent=1)
print(json.dumps(out, indent=1))
