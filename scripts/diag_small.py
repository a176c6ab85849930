"""Where the fixed per-call cost of small levels comes from: event-timed
single calls with and without a preceding L2 flush (read-only 256 MB pass),
compared with trivial torch kernels of the same memory footprint."""
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
flush = torch.zeros(64 * 1024 * 1024, device="cuda")
sink = torch.zeros((), device="cuda")


def t(fn, pre=None, iters=30, graph=True):
    if graph:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        run = g.replay
    else:
        run = fn
    for _ in range(3):
        if pre:
            pre()
        run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        if pre:
            pre()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        run()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return statistics.median(ts), min(ts)


def rd_flush():
    sink.copy_(flush.amax())


def wr_flush():
    flush.zero_()


for W in (512, 2048, 4096):
    x = torch.from_numpy(workloads.uniform_int(W, W, 1)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, W, 1)
    one = torch.zeros(1, device="cuda")
    print(f"== {W}x{W}")
    for name, fn in [("dwt fused", lambda: p.forward(x, y)), ("torch copy", lambda: y.copy_(x)),
                     ("torch add 1 elem", lambda: one.add_(1.0)),
                     ("dwt scheme naive", lambda: p.forward_scheme("nonsep_naive", x, y))]:
        for pre_name, pre in [("warm", None), ("rd-flush", rd_flush), ("wr-flush", wr_flush)]:
            for graph in (True, False):
                med, mn = t(fn, pre, graph=graph)
                print(f"{name:18s} {pre_name:9s} graph={int(graph)}  median {med:7.2f} us  min {mn:7.2f} us")
    p.close()
