"""Parity report (SURVEY.md 8c, c4 comparison procedure): every BASELINE.json
config through the GPU path against the CPU oracle, with the numbers the
tests only assert on -- max-abs error against oracle (i) (fp64 throughout)
and oracle (ii) (fp64 math, each level rounded to fp32), the count of
coefficients that are not bit-identical to (ii), and where the largest error
sits (level, subband, m, n).  Also the inverse (5/3, 9/7) and the 9/7
forward on the config shapes.  Writes JSON lines + a markdown table.

    python tests/report_parity.py [--out profiles/.../parity_report.md]

Test infrastructure (it runs the oracle), hence under tests/; not collected by
pytest (no test_ prefix).
"""
import argparse
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402


def locate(W, H, levels, r, c):
    """(level, subband, m, n) of Mallat position (row r, col c)."""
    w, h = W, H
    for k in range(1, levels + 1):
        wq, hq = (w + 1) // 2, (h + 1) // 2
        if r >= hq or c >= wq or k == levels:
            if r < hq and c < wq:
                return k, "LL", c, r
            band = ("HL" if r < hq else ("LH" if c < wq else "HH"))
            return k, band, c - (wq if c >= wq else 0), r - (hq if r >= hq else 0)
        w, h = wq, hq
    return levels, "LL", c, r


def compare(got, ref_i, ref_ii, W, H, L):
    g = got.astype(np.float64)
    d1 = np.abs(g - ref_i)
    d2 = np.abs(g - ref_ii) if ref_ii is not None else None
    idx = np.unravel_index(int(np.argmax(d1)), d1.shape)
    out = {"max_abs_i": float(d1.max()), "worst_at": locate(W, H, L, int(idx[0]), int(idx[1])),
           "elements": int(g.size)}
    if d2 is not None:
        out["max_abs_ii"] = float(d2.max())
        out["not_bit_exact_vs_ii"] = int(np.count_nonzero(d2))
    return out


def gpu(x, L, wavelet="cdf53", inverse=False, count=1):
    H, W = x.shape[-2:]
    p = dwt2.Plan(W, H, L, max_count=count, wavelet=wavelet)
    t = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    y = (p.inverse(t) if inverse else p.forward(t)).cpu().numpy()
    p.close()
    return y


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "parity_report.md"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    rows = []

    def emit(r):
        rows.append(r)
        print(json.dumps(r), flush=True)

    # forward CDF 5/3, every config (config 5: 4 images of each size, full pyramids)
    for name in ["1", "2", "3", "4", "4b", "5"]:
        cfg = workloads.CONFIGS[name]
        for grp in cfg.groups:
            picks = [0] if name != "5" else [0, grp.count // 3, 2 * grp.count // 3, grp.count - 1]
            for i in picks:
                x = grp.image(i)
                H, W = x.shape
                t0 = time.perf_counter()
                got = gpu(x, cfg.levels)
                x64 = x.astype(np.float64)
                r = compare(got, oracle.forward(x64, cfg.levels), oracle.forward(x64, cfg.levels, round_f32=True),
                            W, H, cfg.levels)
                r.update({"what": "forward cdf53", "config": name, "image": f"{W}x{H} #{i}", "levels": cfg.levels,
                          "seconds": round(time.perf_counter() - t0, 1)})
                emit(r)
    # inverse 5/3 of the oracle's fp32 pyramid, and 9/7 forward / inverse, on configs 2, 4b
    for name in ["2", "4b", "1"]:
        cfg = workloads.CONFIGS[name]
        x = cfg.groups[0].image(0)
        H, W = x.shape
        x64 = x.astype(np.float64)
        y = oracle.forward(x64, cfg.levels, round_f32=True).astype(np.float32)
        got = gpu(y, cfg.levels, inverse=True)
        r = compare(got, oracle.inverse(y.astype(np.float64), cfg.levels),
                    oracle.inverse(y.astype(np.float64), cfg.levels, round_f32=True), W, H, 0)
        r.update({"what": "inverse cdf53", "config": name, "image": f"{W}x{H}", "levels": cfg.levels})
        r.pop("worst_at")
        emit(r)
        got = gpu(x, cfg.levels, wavelet="cdf97")
        r = compare(got, oracle.forward(x64, cfg.levels, wavelet="cdf97"),
                    oracle.forward(x64, cfg.levels, round_f32=True, wavelet="cdf97"), W, H, cfg.levels)
        r.update({"what": "forward cdf97", "config": name, "image": f"{W}x{H}", "levels": cfg.levels})
        emit(r)
        y97 = oracle.forward(x64, cfg.levels, round_f32=True, wavelet="cdf97").astype(np.float32)
        got = gpu(y97, cfg.levels, wavelet="cdf97", inverse=True)
        r = compare(got, oracle.inverse(y97.astype(np.float64), cfg.levels, wavelet="cdf97"),
                    oracle.inverse(y97.astype(np.float64), cfg.levels, round_f32=True, wavelet="cdf97"), W, H, 0)
        r.update({"what": "inverse cdf97", "config": name, "image": f"{W}x{H}", "levels": cfg.levels})
        r.pop("worst_at")
        emit(r)

    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        f.write("# Parity report (GPU vs CPU oracle, B200)\n\n")
        f.write("oracle (i): fp64 throughout; oracle (ii): fp64 arithmetic, every level rounded to fp32 "
                "(the storage type).  Bar (BASELINE.json): max-abs <= 1e-4 vs (i).\n\n")
        f.write("| what | config | image | levels | max abs vs (i) | max abs vs (ii) | not bit-exact vs (ii) "
                "| elements | worst (level, band, m, n) |\n|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            f.write(f"| {r['what']} | {r['config']} | {r['image']} | {r['levels']} | {r['max_abs_i']:.3g} | "
                    f"{r.get('max_abs_ii', float('nan')):.3g} | {r.get('not_bit_exact_vs_ii', '-')} | "
                    f"{r['elements']} | {r.get('worst_at', '-')} |\n")
    print("wrote", args.out)


if __name__ == "__main__":
    main()
