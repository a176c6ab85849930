"""Per-level timeline of one pyramid launch (needs a -DDWT2_PROF build via
DWT2_LIB): for each level of the launch, first tile start and last tile end
relative to the first CTA's work start, tiles, mean blocked time per tile."""
import ctypes
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import _variant  # noqa: E402,F401
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
W = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
L = int(sys.argv[2]) if len(sys.argv) > 2 else 8
n = int(sys.argv[3]) if len(sys.argv) > 3 else 1
x = torch.from_numpy(workloads.smooth_noise(W, W * n, 4).reshape(n, W, W) if n > 1 else workloads.smooth_noise(W, W, 4)).cuda()
y = torch.empty_like(x)
p = dwt2.Plan(W, W, L, max_count=n)
lib = dwt2.lib()
buf = (ctypes.c_ulonglong * (17 * 4))()
for it in range(4):
    lib.dwt2_debug_levels(buf, 1)
    torch.cuda.synchronize()
    p.forward(x, y)
    torch.cuda.synchronize()
    lib.dwt2_debug_levels(buf, 0)
    t0 = buf[16 * 4]
    out = []
    for k in range(16):
        a, b, c, d = buf[4 * k:4 * k + 4]
        if c == 0:
            continue
        out.append(f"L{k}: {(a - t0) / 1e3:6.1f}-{(b - t0) / 1e3:6.1f}us tiles {c} blocked {d / c / 1e3:5.2f}us/tile")
    print(os.environ.get("TAG", ""), f"{W}^2 x{n} L{L} run {it}:", " | ".join(out), flush=True)
