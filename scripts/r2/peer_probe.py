"""One emulated peer-strip step of config 2 on G = 2 ranks, fused and split,
and the NCCL-path step with the exchange stubbed, for an ncu launch list
(per-kernel durations of each form)."""
import sys

import torch

sys.path.insert(0, ".")
if len(sys.argv) > 3:
    from paper_1708_07853_b200 import _build, dwt2 as _d
    _d.use_variant(_build.build_variant(sys.argv[3], {"DWT2_PEER_FENCE_GPU": 1}))
from paper_1708_07853_b200 import distributed as D  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

W = H = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
L = int(sys.argv[2]) if len(sys.argv) > 2 else 1
G = 2
x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
ranks = [D.PeerStripPyramid(W, H, g, G, L, device="cuda") for g in range(G)]
for r in ranks:
    r.connect_local(ranks)
    r.strip.copy_(x[r.r0:r.r1])
for fused in (True, False, True, False):
    D.sequential_step(ranks, fused=fused)
torch.cuda.synchronize()
pyrs = [D.StripPyramid(W, H, g, G, L, device="cuda") for g in range(G)]
plans = [dwt2.StripPlan(W, H, p.r0, p.r1, L) for p in pyrs]
for _ in range(2):
    for p, plan in zip(pyrs, plans):
        D.strip_pyramid_step(p, plan, overlap=True, exchange=lambda k: [])
torch.cuda.synchronize()
print("status", [r.status() for r in ranks])
