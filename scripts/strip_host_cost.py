"""Host cost of one row-strip step (the N > 1 bench path) measured on one GPU:
rank g's strip of config 3 at G = 8 (2048 of 16384 rows), the level kernels
launched exactly as strip_pyramid_step does (interior, boundary), with the
NCCL exchange replaced by a no-op.  If the host time per step exceeds the
GPU time per step, the multi-GPU bench is launch-bound."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1708_07853_b200 import distributed as D  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
for G, L, overlap in [(8, 1, True), (8, 1, False), (2, 1, True), (8, 8, True)]:
    W = H = 16384 if L == 1 else 8192
    g = min(3, G - 2) if G > 2 else 0
    pyr = D.StripPyramid(W, H, g, G, L, device="cuda")
    pyr.strip.copy_(torch.from_numpy(workloads.uniform_int(W, pyr.r1 - pyr.r0, 1)).cuda())
    plan = dwt2.StripPlan(W, H, pyr.r0, pyr.r1, L)
    noop = lambda k: None          # noqa: E731
    for _ in range(20):
        D.strip_pyramid_step(pyr, plan, overlap=overlap, exchange=noop)
    torch.cuda.synchronize()
    K = 200
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    for _ in range(K):
        D.strip_pyramid_step(pyr, plan, overlap=overlap, exchange=noop)
    e1.record()
    t_host = (time.perf_counter() - t0) / K
    torch.cuda.synchronize()
    t_gpu = e0.elapsed_time(e1) / K / 1e3
    # GPU-only time: the same steps replayed from a CUDA graph
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        for _ in range(10):
            D.strip_pyramid_step(pyr, plan, overlap=overlap, exchange=noop)
    gr.replay(); torch.cuda.synchronize()
    e0.record(); gr.replay(); e1.record(); torch.cuda.synchronize()
    t_graph = e0.elapsed_time(e1) / 10 / 1e3
    print(f"G={G} L={L} overlap={overlap}: host enqueue {t_host * 1e6:.1f} us/step, stream time {t_gpu * 1e6:.1f} us/step, "
          f"graph (GPU only) {t_graph * 1e6:.1f} us/step")
    plan.close()
