"""Fused levels 1 + 2 against the oracle (ii), bit for bit, on many sizes
(each level's output rounded to fp32, as the kernels store it)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

rng = np.random.default_rng(3)
cases = [(W, H, L) for W in (4, 5, 6, 7, 8, 9, 13, 16) for H in (4, 5, 6, 7, 8, 9, 11) for L in (2, 3)]
cases += [(120, 64, 2), (121, 64, 2), (239, 240, 2), (240, 241, 3), (241, 239, 2), (244, 100, 2), (480, 37, 2),
          (1000, 777, 3), (1030, 515, 3), (4095, 301, 3), (513, 1025, 4), (2050, 130, 2), (3001, 4095, 3),
          (1537, 1536, 6), (64, 4000, 5), (8193, 300, 4), (4094, 1027, 3), (6, 4099, 2)]
bad = 0
for W, H, L in cases:
    w, h, ok = W, H, True
    for _ in range(L):
        if w < 2 or h < 2:
            ok = False
        w, h = (w + 1) // 2, (h + 1) // 2
    if not ok:
        continue
    x = workloads.uniform_real(W, H, W * 31 + H) if W * H > 4096 else rng.random((H, W)).astype(np.float32) * 255
    p = dwt2.Plan(W, H, L)
    got = p.forward(torch.from_numpy(np.ascontiguousarray(x)).cuda()).cpu().numpy().astype(np.float64)
    p.close()
    ref = oracle.forward(x.astype(np.float64), L, round_f32=True)
    err = np.abs(got - ref)
    n = int((err != 0).sum())
    if n:
        bad += 1
        i = np.unravel_index(np.argmax(err), err.shape)
        print(f"{W}x{H} L{L}: {n} mismatches, max {err.max():.3g} at {i}")
print("cases", len(cases), "bad", bad)
