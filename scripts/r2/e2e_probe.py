"""Where the config-3 e2e time goes: dwt2_forward_host against pure copy
pipelines of the same bytes (pinned host buffers, 1 GiB each way)."""
import time
import torch

import sys, os; sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")); sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_1708_07853_b200 import dwt2

W = H = 16384
N = W * H
hin = torch.empty(N, dtype=torch.float32).pin_memory()
hin.copy_(torch.randint(0, 256, (N,), dtype=torch.int32).float())
hout = torch.empty(N, dtype=torch.float32).pin_memory()
d0 = torch.empty(N, device="cuda")
d1 = torch.empty(N, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
plan = dwt2.Plan(W, H, 1)


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    ts.sort()
    return ts[len(ts) // 2]


def host():
    plan.forward_host(hin.view(H, W), hout.view(H, W))


def chain(nb, dep):
    def f():
        b = N // nb
        for i in range(nb):
            with torch.cuda.stream(s1):
                d0[i * b:(i + 1) * b].copy_(hin[i * b:(i + 1) * b], non_blocking=True)
                e = torch.cuda.Event()
                e.record(s1)
            with torch.cuda.stream(s2):
                if dep:
                    s2.wait_event(e)
                hout[i * b:(i + 1) * b].copy_(d1[i * b:(i + 1) * b], non_blocking=True)
    return f


for name, fn in [("forward_host", host), ("copies16", chain(16, False)), ("dep16", chain(16, True)),
                 ("dep64", chain(64, True)), ("forward_host", host)]:
    t = timed(fn)
    print(f"{name:13s} {t*1e3:7.2f} ms  {N / t / 1e9:6.2f} Gpix/s", flush=True)
