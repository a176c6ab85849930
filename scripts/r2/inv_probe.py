"""Inverse 5/3 timing on odd-pitch (plain-load kernel) and aligned shapes: K = 10
graph-captured calls (scripts/_timing.py), fraction of copy per level-1 bytes."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
out = []
for W, H, L in [(8193, 8193, 1), (8193, 8193, 8), (4095, 3001, 3), (16383, 8191, 1), (8192, 8192, 1)]:
    x = torch.from_numpy(workloads.smooth_noise(W, H, 4)).cuda()
    p = dwt2.Plan(W, H, L)
    y = p.forward(x).clone()
    r = torch.empty_like(x)
    us = time_calls(lambda q: p.inverse(q[0], q[1]), [(y, r)], 10)
    out.append(f"{W}x{H} L{L} {us:.1f}us" + (f" ({8 * W * H / us / 1e3 / 6535:.3f})" if L == 1 else ""))
    p.close()
print(os.environ.get("TAG", ""), " | ".join(out), flush=True)
