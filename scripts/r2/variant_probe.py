"""One-level and pyramid timings (K = 20 calls in one graph, bench.py's buffer
protocol) for a library build given as argv[1] ("product" = the in-tree one)."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from paper_1708_07853_b200 import dwt2  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "product"
if tag != "product":
    dwt2.use_variant(tag)
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

for name, W, H, L, npairs in [("config 2", 4096, 4096, 1, 3), ("16384x2048", 16384, 2048, 1, 2),
                              ("8192^2", 8192, 8192, 1, 1), ("config 3", 16384, 16384, 1, 1),
                              ("config 4", 8192, 8192, 8, 1)]:
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    pairs = [(x.clone(), torch.empty_like(x)) for _ in range(npairs)]
    p = dwt2.Plan(W, H, L)
    us = time_calls(lambda q: p.forward(q[0], q[1]), pairs, 20)
    print(f"{tag.split('/')[-1]} {name}: {us:.1f} us", flush=True)
    p.close()
    del pairs, x
