"""Why a config-3 strip at G = 2 costs more than half the 1-GPU step: the
same rows as a plain 16384 x 8192 image, and the strip's launches alone."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import distributed as D  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
W = 16384
for Hs in (8192, 8194, 4096, 2048):
    x = torch.from_numpy(workloads.uniform_int(W, Hs, 1)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, Hs, 1)
    print(f"plain {W}x{Hs}: {time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 10):.1f} us")
    p.close()
H = 16384
x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
noop = lambda k: None  # noqa: E731
for G in (2, 4, 8):
    pyr = D.StripPyramid(W, H, 0, G, 1, device="cuda")
    pyr.strip.copy_(x[pyr.r0:pyr.r1])
    plan = dwt2.StripPlan(W, H, pyr.r0, pyr.r1, 1)
    h = plan.handle
    b = pyr.bufs[0]
    for part, nm in ((dwt2.DWT2_STRIP_ALL, "ALL"), (dwt2.DWT2_STRIP_INTERIOR, "INTERIOR"), (dwt2.DWT2_STRIP_BOUNDARY, "BOUNDARY")):
        us = time_calls(lambda q: dwt2.dwt2_forward_strip_level(h, 0, b.data_ptr(), b.stride(0), 0, 0, pyr.out.data_ptr(),
                                                                part, torch.cuda.current_stream().cuda_stream), [(None,)], 10)
        print(f"G={G} rank 0 ({pyr.r1 - pyr.r0} rows): {nm} {us:.1f} us")
    plan.close()
