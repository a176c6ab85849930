"""Needs scripts/experiments/level_dataflow_pdl.patch applied (not shipped).
Dataflow between the level launches of a multi-level forward (dwt2.cu
"Dataflow") against the same build with it off (a -DDWT2_TUNING variant run
with DWT2_DATAFLOW=0): configs 4, 4b, a config-5 group and 4096^2 at 3 levels,
K = 20 calls in one CUDA graph, and each output compared with the product's.
Round-2 bound measured before it existed: levels >= 2 skipping
griddepcontrol.wait altogether (wrong results) gave config 4 140.4 -> 129.8 us,
4b 150.5 -> 133.4, the config-5 2048^2 x 32 group 255.5 -> 241.1, 4096^2 L3
38.9 -> 34.1."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import _build, dwt2  # noqa: E402

mode = sys.argv[1] if len(sys.argv) > 1 else "product"
if mode == "nodf":
    os.environ["DWT2_DATAFLOW"] = "0"
    dwt2.use_variant(_build.build_variant("tuning", {"DWT2_TUNING": 1}))
elif mode.startswith("from"):                   # from<k>: level k is the first dataflow producer
    os.environ["DWT2_DF_FROM"] = mode[4:]
    dwt2.use_variant(_build.build_variant("tuning", {"DWT2_TUNING": 1}))
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for name, W, H, L, n in [("config 4", 8192, 8192, 8, 1), ("config 4b", 8193, 8193, 8, 1),
                         ("config 5 group 2048^2 x 32", 2048, 2048, 3, 32),
                         ("config 5 group 4095x3001 x 8", 4095, 3001, 3, 8), ("4096^2 L3", 4096, 4096, 3, 1)]:
    x = torch.from_numpy(workloads.smooth_noise(W, H, 1)).cuda()
    if n > 1:
        x = x.expand(n, H, W).contiguous()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, L, max_count=n)
    us = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 20)
    print(f"{mode} {name}: {us:.1f} us", flush=True)
    p.close()
