"""Grouped tail kernel (tail.cu dwt_ptail_kernel, tuning build knobs
DWT2_TAIL_GROUPED / DWT2_PT_*): forward pyramids against the oracle -- 5/3 bit
for bit vs oracle (ii), 9/7 within 1e-4 of oracle (i) -- over odd and even
sizes, all level counts and batches, with every level in the tail
(DWT2_TAIL_QUADS / DWT2_K2_TAIL_QUADS large) or the default split."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)) + "/..")
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)) + "/../..")
import _variant  # noqa: E402,F401
import oracle  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402


def lmax(W, H):
    L = 0
    while W >= 2 and H >= 2:
        W, H, L = (W + 1) // 2, (H + 1) // 2, L + 1
    return L


rng = np.random.default_rng(int(os.environ.get("SEED", "5")))
shapes = [(2, 2), (3, 2), (2, 3), (3, 3), (5, 7), (6, 6), (9, 10), (33, 17), (64, 64), (100, 37), (255, 257),
          (256, 256), (257, 255), (300, 212), (513, 511), (1024, 1024), (1023, 1025)]
shapes += [(int(rng.integers(2, 1500)), int(rng.integers(2, 1500))) for _ in range(int(os.environ.get("NRAND", "25")))]
bad = 0
n = 0
for wav in ("cdf53", "cdf97"):
    for (W, H) in shapes:
        Ls = sorted(set([1, 2, lmax(W, H), max(1, lmax(W, H) - 2)]))
        for L in Ls:
            if L > lmax(W, H):
                continue
            count = int(rng.choice([1, 1, 2, 3]))
            xs = np.stack([workloads.uniform_real(W, H, W * 7 + H + i) for i in range(count)])
            plan = dwt2.Plan(W, H, L, max_count=count, wavelet=wav)
            got = plan.forward(torch.from_numpy(xs if count > 1 else xs[0]).cuda()).cpu().numpy().reshape(count, H, W)
            plan.close()
            for i in range(count):
                n += 1
                if wav == "cdf53":
                    ref = oracle.forward(xs[i].astype(np.float64), L, round_f32=True)
                    d = np.abs(got[i].astype(np.float64) - ref)
                    ok = not d.any()
                else:
                    ref = oracle.forward(xs[i].astype(np.float64), L, round_f32=False, wavelet="cdf97")
                    d = np.abs(got[i].astype(np.float64) - ref)
                    ok = d.max() <= 1e-4
                if not ok:
                    bad += 1
                    if bad < 20:
                        print(f"MISMATCH {wav} {W}x{H} L{L} count {count} img {i}: {int(np.count_nonzero(d))} off, max {d.max()}", flush=True)
print(f"ptail_check: {n} images, {bad} bad", flush=True)
