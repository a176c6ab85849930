"""Pyramid-launch probe: time the multi-level forward of config 4 (8192^2, 8
levels), 4b and one config-5 group (64 x 2048^2, 3 levels) as K graph-captured
calls (scripts/_timing.py protocol).  With a -DDWT2_TUNING build (DWT2_LIB),
DWT2_PYRAMID=0 gives the per-level launches for comparison and DWT2_PYR_*
change the pyramid tile policy."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
res = []
for name, W, H, L, n in [("c4", 8192, 8192, 8, 1), ("c4b", 8193, 8193, 8, 1), ("c5g", 2048, 2048, 3, 64)]:
    if n == 1:
        x = torch.from_numpy(workloads.smooth_noise(W, H, 4)).cuda()
    else:
        x = torch.from_numpy(workloads.uniform_int(W, H * n, 5).reshape(n, H, W)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, L, max_count=n)
    us = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 20)
    res.append(f"{name} {us:.1f}us")
    p.close()
print(os.environ.get("TAG", ""), " ".join(res), flush=True)
