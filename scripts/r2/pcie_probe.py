"""Pinned host <-> device copy rates on the box (the e2e bound): H2D alone,
D2H alone, both at once on two streams, for 1 GiB, and in 16 / 64 bands."""
import time
import torch

N = 1 << 28                      # 1 GiB of fp32
hin = torch.empty(N, dtype=torch.float32).pin_memory()
hout = torch.empty(N, dtype=torch.float32).pin_memory()
d0 = torch.empty(N, device="cuda")
d1 = torch.empty(N, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts)


def h2d():
    with torch.cuda.stream(s1):
        d0.copy_(hin, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        hout.copy_(d1, non_blocking=True)


def both():
    h2d()
    d2h()


def banded(nb):
    def f():
        b = N // nb
        for i in range(nb):
            with torch.cuda.stream(s1):
                d0[i * b:(i + 1) * b].copy_(hin[i * b:(i + 1) * b], non_blocking=True)
            with torch.cuda.stream(s2):
                hout[i * b:(i + 1) * b].copy_(d1[i * b:(i + 1) * b], non_blocking=True)
    return f


GB = N * 4 / 1e9
for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both), ("both16", banded(16)), ("both64", banded(64))]:
    t = timed(fn)
    print(f"{name:7s} {t*1e3:7.2f} ms  {GB / t:6.1f} GB/s per direction", flush=True)
print("device", torch.cuda.get_device_name(0))
