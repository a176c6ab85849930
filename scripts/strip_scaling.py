"""Per-rank GPU time of the row-strip step (the N > 1 bench path) for G = 1,
2, 4, 8, measured on one GPU with the NCCL exchange replaced by a no-op:
rank g's strip_pyramid_step (interior + boundary launches per level) replayed
from a CUDA graph.  The max over the ranks measured, against the 1-GPU step,
bounds the strong-scaling efficiency the exchange can only lower:
E(G) <= T(1) / (G * max_g T_g(G))."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import distributed as D  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
noop = lambda k: None  # noqa: E731
for name, W, H, L in [("config 3", 16384, 16384, 1), ("config 4", 8192, 8192, 8)]:
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, L)
    t1 = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 10)
    p.close()
    print(f"{name}: G=1 {t1:7.1f} us/step")
    for G in (2, 4, 8):
        worst = 0.0
        ranks = sorted({0, min(1, G - 1), G - 1})
        per = []
        for g in ranks:
            pyr = D.StripPyramid(W, H, g, G, L, device="cuda")
            pyr.strip.copy_(x[pyr.r0:pyr.r1])
            plan = dwt2.StripPlan(W, H, pyr.r0, pyr.r1, L)
            us = time_calls(lambda q: D.strip_pyramid_step(pyr, plan, overlap=True, exchange=noop), [(None,)], 10)
            per.append(f"rank {g}: {us:.1f}")
            worst = max(worst, us)
            plan.close()
            del pyr
        print(f"{name}: G={G} max {worst:7.1f} us/step ({', '.join(per)}); "
              f"E(G) <= {t1 / (G * worst):.2f}")
