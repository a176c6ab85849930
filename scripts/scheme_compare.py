"""The paper's scheme comparison (section 4, Fig. 6) on
B200: every scheme of csrc/schemes.cu plus the fused product kernel, one
level of the forward 2-D CDF 5/3 DWT on integer-valued images of edge
1024 .. 16384 (protocol of scripts/_timing.py: K calls in one CUDA graph,
distinct input/output pairs for small sizes, L2 flushed before the replay).

A step boundary is a kernel boundary, so the schemes differ in HBM round
trips: algorithmic bytes per pixel = 8 (1 step, fused / naive), 16 (2 steps:
Eq. 4 convolution, Eq. 5 lifting, Fig. 3 adapted), 26 (Eq. 3, 4 steps:
8 + 3 x 6, the in-place separable steps read 4 B and write 2 B per pixel).

Every scheme's output is first checked bit-exact against the fused kernel
(integer inputs, one level: all schemes are exact).  Prints one JSON line per
(size, scheme) and a markdown table at the end.

    python scripts/scheme_compare.py [--sizes 1024,2048,...] [--iters 30]
"""
import argparse
import json
import os
import statistics
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from _timing import n_pairs, time_calls  # noqa: E402

BYTES = {"fused": 8, "fused_literal": 8, "fused_adapted": 8, "nonsep_naive": 8, "nonsep_lifting": 16,
         "nonsep_adapted": 16, "sep_conv": 16, "sep_lifting": 26}
PAPER = {"fused": "Eq. 5 fused (product)", "fused_literal": "Eq. 5 fused, literal 24-MAC operators",
         "fused_adapted": "Fig. 3 adapted, fused", "nonsep_naive": "Eq. 5, 1 plain kernel",
         "nonsep_lifting": "Eq. 5 non-separable lifting", "nonsep_adapted": "Fig. 3 adapted non-separable",
         "sep_conv": "Eq. 4 separable convolution", "sep_lifting": "Eq. 3 separable lifting"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="1024,2048,4096,8192,16384")
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "scheme_compare.json"))
    args = ap.parse_args()
    torch.cuda.set_device(0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    rows = []
    for edge in [int(s) for s in args.sizes.split(",")]:
        x = torch.from_numpy(workloads.uniform_int(edge, edge, 3)).cuda()
        plan = dwt2.Plan(edge, edge, 1)
        ref = plan.forward(x)
        torch.cuda.synchronize()
        npairs = n_pairs(8 * edge * edge, args.iters)
        pairs = [(x if i == 0 else x.clone(), torch.empty_like(x)) for i in range(npairs)]
        for scheme in BYTES:
            out = torch.empty_like(x)
            plan.forward_scheme(scheme, x, out)
            torch.cuda.synchronize()
            exact = bool(torch.equal(out, ref))
            us = time_calls(lambda p, s=scheme: plan.forward_scheme(s, p[0], p[1]), pairs, args.iters)
            px = edge * edge
            r = {"edge": edge, "scheme": scheme, "paper": PAPER[scheme],
                 "steps": dwt2.dwt2_scheme_steps(dwt2.SCHEMES[scheme]), "us": us,
                 "gpix_s": px / us / 1e3, "ns_per_pel": us * 1e3 / px,
                 "algo_bytes_per_px": BYTES[scheme], "algo_gbs": BYTES[scheme] * px / us / 1e3,
                 "frac_of_copy": BYTES[scheme] * px / us / 1e3 / peak, "bit_exact_vs_fused": exact}
            rows.append(r)
            print(json.dumps(r), flush=True)
        del pairs
        plan.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out, "w") as f:
        json.dump({"peak_gbs": peak, "rows": rows}, f, indent=1)
    # markdown table: time per scheme and speed-up of the fused kernel
    print("\n| edge | " + " | ".join(BYTES) + " |")
    print("|---" * (len(BYTES) + 1) + "|")
    for edge in sorted({r["edge"] for r in rows}):
        cells = []
        for s in BYTES:
            r = next(r for r in rows if r["edge"] == edge and r["scheme"] == s)
            cells.append(f"{r['us']:.1f} us ({r['frac_of_copy']:.2f})")
        print(f"| {edge} | " + " | ".join(cells) + " |")


if __name__ == "__main__":
    main()
