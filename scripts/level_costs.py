"""Marginal cost of each pyramid level in the real launch sequence (CUDA
graph, PDL between levels): time Plan(W, H, L) for L = 1..Lmax and print
the differences.  python scripts/level_costs.py [W H Lmax]."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import n_pairs, time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
H = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
Lmax = int(sys.argv[3]) if len(sys.argv) > 3 else 8
WAV = sys.argv[4] if len(sys.argv) > 4 else "cdf53"
OP = sys.argv[5] if len(sys.argv) > 5 else "forward"
K = 20
x = torch.from_numpy(workloads.smooth_noise(W, H, 4) if hasattr(workloads, "smooth_noise")
                     else workloads.GENERATORS["smooth"](W, H, 4)).cuda()
np_ = n_pairs(8 * W * H, K)
pairs = [(x.clone() if i else x, torch.empty_like(x)) for i in range(np_)]
prev = 0.0
w, h = W, H
for L in range(1, Lmax + 1):
    p = dwt2.Plan(W, H, L, wavelet=WAV)
    if OP == "inverse":
        ipairs = [(p.forward(q[0]).clone(), q[1]) for q in pairs]
        us = time_calls(lambda q: p.inverse(q[0], q[1]), ipairs, K)
    else:
        us = time_calls(lambda q: p.forward(q[0], q[1]), pairs, K)
    print(f"L={L}: {us:8.2f} us total, level {L} ({w}x{h}, {8 * w * h / 1e6:7.2f} MB): +{us - prev:6.2f} us")
    prev = us
    w, h = (w + 1) // 2, (h + 1) // 2
    p.close()
