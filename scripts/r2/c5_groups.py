"""Config 5's two groups timed separately (K = 10 batched calls in one graph)
for a library build given as argv[1] ("product" = the in-tree one)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import dwt2  # noqa: E402

if len(sys.argv) > 1 and sys.argv[1] != "product":
    dwt2.use_variant(sys.argv[1])
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for W, H, n, L in [(2048, 2048, 256, 3), (4095, 3001, 32, 3), (2048, 2048, 256, 1), (4095, 3001, 32, 1)]:
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda().expand(n, H, W).contiguous()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, L, max_count=n)
    us = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 10)
    print(f"{sys.argv[1] if len(sys.argv) > 1 else 'product'} {n}x{W}x{H} L{L}: {us:.1f} us", flush=True)
    p.close()
    del x, y
