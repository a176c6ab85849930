"""Inverse small levels: the small-level inverse kernel (tail.cu
dwt_small_inv_kernel) for levels of <= DWT2_INV_SMALL_QUADS quads against the
inverse level kernels; argv[1] = threshold ("product" = shipped), K = 20 calls
in one graph, pyramid input as bench.py builds it."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import _build, dwt2  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "product"
if mode != "product":
    os.environ["DWT2_INV_SMALL_QUADS"] = mode
    dwt2.use_variant(_build.build_variant("tuning", {"DWT2_TUNING": 1}))
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for name, W, H, L, wav in [("5/3 config 4", 8192, 8192, 8, "cdf53"), ("5/3 config 4b", 8193, 8193, 8, "cdf53"),
                           ("9/7 config 4", 8192, 8192, 8, "cdf97"), ("5/3 1024^2 L1", 1024, 1024, 1, "cdf53"),
                           ("9/7 1024^2 L1", 1024, 1024, 1, "cdf97")]:
    x = torch.from_numpy(workloads.smooth_noise(W, H, 1)).cuda()
    p = dwt2.Plan(W, H, L, wavelet=wav)
    y = p.forward(x).clone()
    npairs = 20 if W * H * 8 < 2 * 126e6 else 1
    pairs = [(y.clone(), torch.empty_like(y)) for _ in range(npairs)]
    us = time_calls(lambda q: p.inverse(q[0], q[1]), pairs, 20)
    print(f"inv_small={mode} {name}: {us:.1f} us", flush=True)
    p.close()
