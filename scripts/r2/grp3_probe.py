"""Large levels with pitches that are not a multiple of 16 bytes: the 3-stage
row-grouped TMA kernel (product) against the 2-stage one (a -DDWT2_TUNING
variant with DWT2_LARGE_S3G=0; argv[1] = "product" or "off").  K = 10 calls in
one CUDA graph."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import _build, dwt2  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "product"
if mode == "off":
    os.environ["DWT2_LARGE_S3G"] = "0"
    dwt2.use_variant(_build.build_variant("tuning", {"DWT2_TUNING": 1}))
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for name, W, H, L, n in [("4095x3001 x 32 L3", 4095, 3001, 3, 32), ("4095x3001 x 32 L1", 4095, 3001, 1, 32),
                         ("16383x16383 L1", 16383, 16383, 1, 1), ("8193^2 L8", 8193, 8193, 8, 1),
                         ("16382x8191 L1", 16382, 8191, 1, 1)]:
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    if n > 1:
        x = x.expand(n, H, W).contiguous()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, L, max_count=n)
    us = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 10)
    print(f"s3g={mode} {name}: {us:.1f} us", flush=True)
    p.close()
    del x, y
