"""Throughput of the GPU inverse next to the forward,
on the BASELINE.json config shapes: per config, device-resident inputs,
protocol of scripts/_timing.py (K calls in one CUDA graph, distinct buffer
pairs for small sizes, L2 flushed before the timed replay).  Algorithmic bytes as the forward: 8 B per pixel per
level.  Also checks inverse(forward(x)) == x on the integer configs.

    python scripts/inverse_bench.py [--iters 30]
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=20)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    for name in ["1", "2", "3", "4", "4b"]:
        cfg = workloads.CONFIGS[name]
        g0 = cfg.groups[0]
        x = torch.from_numpy(g0.image(0)).cuda()
        plan = dwt2.Plan(g0.width, g0.height, cfg.levels)
        y = plan.forward(x)
        rec = torch.empty_like(x)
        plan.inverse(y, rec)
        torch.cuda.synchronize()
        err = float((rec - x).abs().max())
        npairs = n_pairs(8 * x.numel(), args.iters)
        fwd_pairs = [(x if i == 0 else x.clone(), torch.empty_like(x)) for i in range(npairs)]
        inv_pairs = [(y if i == 0 else y.clone(), torch.empty_like(x)) for i in range(npairs)]
        t_fwd = time_calls(lambda p: plan.forward(p[0], p[1]), fwd_pairs, args.iters)
        t_inv = time_calls(lambda p: plan.inverse(p[0], p[1]), inv_pairs, args.iters)
        px = g0.width * g0.height
        algo = 8 * workloads.level_pixels(g0.width, g0.height, cfg.levels)
        p1 = dwt2.Plan(g0.width, g0.height, 1)
        inv1_pairs = [(p1.forward(a), torch.empty_like(x)) for a, _ in fwd_pairs]
        t_inv1 = time_calls(lambda p: p1.inverse(p[0], p[1]), inv1_pairs, args.iters)
        p1.close()
        r = {"config": name, "levels": cfg.levels, "size": f"{g0.width}x{g0.height}",
             "forward_us": t_fwd, "inverse_us": t_inv,
             "forward_gpix_s": px / t_fwd / 1e3, "inverse_gpix_s": px / t_inv / 1e3,
             "inverse_algo_gbs": algo / t_inv / 1e3, "inverse_level1_us": t_inv1,
             "inverse_level1_frac_of_copy": 8 * px / t_inv1 / 1e3 / peak,
             "round_trip_max_abs": err, "buffer_pairs": npairs}
        print(json.dumps(r), flush=True)
        del fwd_pairs, inv_pairs, inv1_pairs
        plan.close()


if __name__ == "__main__":
    main()
