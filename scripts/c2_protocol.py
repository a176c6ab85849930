"""Config 2 per-call time under different cold-cache protocols: K graph-
captured calls cycling over P distinct buffer pairs (P = 2, 4, 10, 20), with
one L2 flush before the replay; and the single-pair warm number."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
W = H = 4096
x = torch.from_numpy(workloads.GENERATORS["smooth"](W, H, 2)).cuda()
p = dwt2.Plan(W, H, 1)
for P in (1, 2, 4, 10, 20):
    pairs = [(x.clone(), torch.empty_like(x)) for _ in range(P)]
    for K in (20,):
        us = time_calls(lambda q: p.forward(q[0], q[1]), pairs, K)
        print(f"pairs {P:2d}, K {K}: {us:6.1f} us/call ({8 * W * H / us / 1e3 / 6535:.3f} of copy)")
    del pairs
