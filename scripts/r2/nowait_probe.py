"""Upper bound of overlapping a level's drain with the next level's start:
a probe build whose level launches >= 2 skip griddepcontrol.wait at entry
(their results are WRONG -- timing only) against the product build, config 4,
4b and one config-5 group (K = 20 calls in one CUDA graph)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import _build, dwt2  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] == "nowait":
    dwt2.use_variant(_build.build_variant("nowait", {"DWT2_PROBE_NOWAIT": 1}))
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for name, W, H, L, n in [("config 4", 8192, 8192, 8, 1), ("config 4b", 8193, 8193, 8, 1),
                         ("config 5 group 2048^2 x 32", 2048, 2048, 3, 32), ("4096^2 L3", 4096, 4096, 3, 1)]:
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    if n > 1:
        x = x.expand(n, H, W).contiguous()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, L, max_count=n)
    us = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 20)
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'product'} {name}: {us:.1f} us", flush=True)
    p.close()
