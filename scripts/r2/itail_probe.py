"""Inverse tail vs inverse level kernels on small pyramids (graph of K calls):
per-call time for W^2 images with L levels, DWT2_ITAIL_QUADS / DWT2_K2_ITAIL_QUADS
selecting how many coarse levels run in the inverse tail (tuning build)."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
out = []
for W, L, wav in [(256, 1, "cdf53"), (256, 3, "cdf53"), (1024, 5, "cdf53"), (256, 1, "cdf97"), (256, 3, "cdf97"),
                  (1024, 5, "cdf97")]:
    x = torch.from_numpy(workloads.smooth_noise(W, W, 4)).cuda()
    p = dwt2.Plan(W, W, L, wavelet=wav)
    y = p.forward(x).clone()
    r = torch.empty_like(x)
    us = time_calls(lambda q: p.inverse(q[0], q[1]), [(y, r)], 20)
    out.append(f"{wav} {W}^2 L{L} {us:.1f}us")
    p.close()
print(os.environ.get("TAG", ""), " | ".join(out), flush=True)
