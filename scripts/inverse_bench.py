"""Throughput of the GPU inverse next to the forward,
on the BASELINE.json config shapes: per config, device-resident input, CUDA
graph of one call, L2 flushed before every timed iteration for inputs that
fit in L2, median of N.  Algorithmic bytes as the forward: 8 B per pixel per
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


def timed(fn, flush, iters):
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    # K (flush + call) back to back minus K flushes alone (event ticks are 2.048 us)
    def run(k, with_call):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(k):
            if flush is not None:
                flush.amax()
            if with_call:
                g.replay()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) * 1e3
    ts = [(run(iters, True) - run(iters, False)) / iters for _ in range(5)]
    return statistics.median(ts)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=30)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    flush_buf = torch.zeros(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
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
        flush = flush_buf if x.numel() * 4 <= 126e6 else None
        t_fwd = timed(lambda: plan.forward(x, y), flush, args.iters)
        t_inv = timed(lambda: plan.inverse(y, rec), flush, args.iters)
        px = g0.width * g0.height
        algo = 8 * workloads.level_pixels(g0.width, g0.height, cfg.levels)
        # level-1 inverse alone (the dominant launch)
        p1 = dwt2.Plan(g0.width, g0.height, 1)
        y1 = p1.forward(x)
        r1 = torch.empty_like(x)
        t_inv1 = timed(lambda: p1.inverse(y1, r1), flush, args.iters)
        p1.close()
        r = {"config": name, "levels": cfg.levels, "size": f"{g0.width}x{g0.height}",
             "forward_us": t_fwd, "inverse_us": t_inv,
             "forward_gpix_s": px / t_fwd / 1e3, "inverse_gpix_s": px / t_inv / 1e3,
             "inverse_algo_gbs": algo / t_inv / 1e3, "inverse_level1_us": t_inv1,
             "inverse_level1_frac_of_copy": 8 * px / t_inv1 / 1e3 / peak,
             "round_trip_max_abs": err, "l2": "flushed" if flush is not None else "input > L2"}
        print(json.dumps(r), flush=True)
        plan.close()


if __name__ == "__main__":
    main()
