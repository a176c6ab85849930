# Test tooling (runs the oracle), kept under tests/ (not collected: no test_ prefix).
"""Locate parity failures: for each (W, H, L) print max error per level/band."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
import oracle
from paper_1708_07853_b200 import dwt2, workloads

cases = [(1030, 515, 1), (1030, 515, 2), (1030, 515, 3), (1032, 515, 1), (515, 300, 1), (516, 300, 1),
         (1024, 1024, 2), (2050, 130, 1), (2048, 37, 1), (600, 40, 1), (520, 40, 1), (300, 40, 1)]
for W, H, L in cases:
    x = workloads.uniform_int(W, H, 5)
    p = dwt2.Plan(W, H, L)
    out = p.forward(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    ref = oracle.forward(x.astype(np.float64), L, round_f32=True)
    d = np.abs(out - ref)
    bad = np.argwhere(d > 0)
    print(f"{W}x{H} L{L}: max {d.max():.4g} nbad {len(bad)}", bad[:5].tolist() if len(bad) else "")
