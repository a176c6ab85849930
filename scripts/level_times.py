"""Marginal cost of each level of a pyramid: T(L levels) - T(L-1), CUDA-graph replays."""
import sys
import torch
sys.path.insert(0, '.')
from paper_1708_07853_b200 import dwt2, workloads

def timed(W, H, L, x, out, reps=50):
    p = dwt2.Plan(W, H, L)
    p.forward(x, out); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        p.forward(x, out)
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): g.replay()
    e1.record(); torch.cuda.synchronize()
    p.close()
    return e0.elapsed_time(e1) / reps * 1e3

for (W, H, LMAX) in [(8192, 8192, 8), (2048, 2048, 3)]:
    x = torch.from_numpy(workloads.smooth_noise(W, H, 4)).cuda()
    out = torch.empty_like(x)
    prev = 0.0
    for L in range(1, LMAX + 1):
        t = timed(W, H, L, x, out)
        w, h = W, H
        for _ in range(L - 1): w, h = (w + 1) // 2, (h + 1) // 2
        print(f"{W}x{H} L={L}: total {t:8.1f} us   level {L} ({w}x{h}) +{t - prev:7.1f} us  ({8*w*h/max(t-prev,1e-3)/1e3:7.0f} GB/s)")
        prev = t
