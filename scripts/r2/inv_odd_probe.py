"""Inverse of odd-width images (Mallat pitch not 16-byte aligned: the plain-load
inverse level kernel) against the small-level inverse kernel on every level
(-DDWT2_TUNING variant, DWT2_INV_SMALL_QUADS_ODD = argv[1]; "product" = shipped)."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import _build, dwt2  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "product"
if mode != "product":
    os.environ["DWT2_INV_SMALL_QUADS_ODD"] = mode
    dwt2.use_variant(_build.build_variant("tuning", {"DWT2_TUNING": 1}))
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for name, W, H, L, n in [("4b 8193^2 L8", 8193, 8193, 8, 1), ("8193^2 L1", 8193, 8193, 1, 1),
                         ("4095x3001 x 32 L3", 4095, 3001, 3, 32), ("4095x3001 L1", 4095, 3001, 1, 1)]:
    x = torch.from_numpy(workloads.smooth_noise(W, H, 1)).cuda()
    if n > 1:
        x = x.expand(n, H, W).contiguous()
    p = dwt2.Plan(W, H, L, max_count=n)
    y = p.forward(x).clone()
    npairs = 1 if W * H * n * 8 >= 2 * 126e6 else 3
    pairs = [(y.clone(), torch.empty_like(y)) for _ in range(npairs)]
    us = time_calls(lambda q: p.inverse(q[0], q[1]), pairs, 10)
    print(f"inv_odd={mode} {name}: {us:.1f} us", flush=True)
    p.close()
    del x, y, pairs
