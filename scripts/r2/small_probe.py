"""Small single levels: the small-level kernel (product) against the level
kernel (a -DDWT2_TUNING variant with DWT2_SMALL_QUADS=0), K = 20 calls in one
CUDA graph, each call on its own buffer pair after an L2 flush (bench.py's
config-1 protocol); plus config 4 (levels 4-5 of 1024^2 / 512^2 input become
small at larger thresholds: DWT2_SMALL_QUADS=2^18 in a second variant run)."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import _build, dwt2  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "product"
if mode != "product":
    os.environ["DWT2_SMALL_QUADS"] = mode
    os.environ["DWT2_SMALL_QUADS_LL"] = os.environ.get("LLQ", "262144")
    dwt2.use_variant(_build.build_variant("tuning", {"DWT2_TUNING": 1}))
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

CASES = [("config 1", 512, 512, 1), ("256^2", 256, 256, 1), ("1024^2", 1024, 1024, 1),
         ("config 4", 8192, 8192, 8), ("config 4b", 8193, 8193, 8)]
if len(sys.argv) > 2 and sys.argv[2] == "mid":
    CASES = [("2048^2", 2048, 2048, 1), ("config 2", 4096, 4096, 1), ("16384x2048", 16384, 2048, 1),
             ("8192^2", 8192, 8192, 1), ("config 4", 8192, 8192, 8)]
for name, W, H, L in CASES:
    K = 20
    npairs = K if W * H * 8 < 2 * 126e6 else 1
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    pairs = [(x.clone(), torch.empty_like(x)) for _ in range(npairs)]
    p = dwt2.Plan(W, H, L)
    us = time_calls(lambda q: p.forward(q[0], q[1]), pairs, K)
    print(f"small_quads={mode} {name}: {us:.2f} us", flush=True)
    p.close()
