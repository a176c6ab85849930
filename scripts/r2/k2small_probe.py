"""CDF 9/7 (K = 2) small levels: the radius-4 small-level kernel (tail.cu
dwt_small4_kernel) for levels of <= DWT2_K2_SMALL_QUADS quads against the K = 2
level kernel; config 4 (9/7) and single levels, K = 20 calls in one graph
(-DDWT2_TUNING variant; argv[1] = the threshold, "product" = the shipped one)."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import _build, dwt2  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "product"
if mode != "product":
    os.environ["DWT2_K2_SMALL_QUADS"] = mode
    dwt2.use_variant(_build.build_variant("tuning", {"DWT2_TUNING": 1}))
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for name, W, H, L in [("9/7 config 4", 8192, 8192, 8), ("9/7 config 4b", 8193, 8193, 8),
                      ("9/7 2048^2 L1", 2048, 2048, 1), ("9/7 1024^2 L1", 1024, 1024, 1), ("9/7 512^2 L1", 512, 512, 1)]:
    K = 20
    npairs = K if W * H * 8 < 2 * 126e6 else 1
    x = torch.from_numpy(workloads.smooth_noise(W, H, 1)).cuda()
    pairs = [(x.clone(), torch.empty_like(x)) for _ in range(npairs)]
    p = dwt2.Plan(W, H, L, wavelet="cdf97")
    us = time_calls(lambda q: p.forward(q[0], q[1]), pairs, K)
    print(f"k2_small={mode} {name}: {us:.2f} us", flush=True)
    p.close()
