"""Single-level timing of W x H (K graph-captured calls): with a tuning build,
DWT2_PYR_MIN=1 runs the level as a one-level pyramid launch (the pyramid
kernel's per-tile overhead against the level kernel), DWT2_PYR_PUBLAST=1 adds
the readiness publishes."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
a = [int(v) for v in sys.argv[1:]] or [16384, 16384, 8192, 8192, 4096, 4096]
out = []
for W, H in zip(a[0::2], a[1::2]):
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, 1)
    us = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 10)
    out.append(f"{W}x{H} {us:.1f}us ({8 * W * H / us / 1e3 / 6535:.3f})")
    p.close()
print(os.environ.get("TAG", ""), " | ".join(out), flush=True)
