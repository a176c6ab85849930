"""PCIe probe: raw pinned H2D / D2H bandwidth of 1 GiB, both directions at
once, and dwt2_forward_host end to end for config 3 (16384^2) -- the bound
of bench.py's e2e number."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

n = 16384 * 16384
h = torch.empty(n, dtype=torch.float32).pin_memory()
h2 = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
d2 = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in [("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h2.copy_(d2, non_blocking=True))]:
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    print(f"{name}: {3 * n * 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s")
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(3):
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print(f"H2D || D2H: {3 * 2 * n * 4 / (time.perf_counter() - t) / 1e9:.1f} GB/s total")
x = torch.from_numpy(workloads.uniform_int(16384, 16384, 3)).pin_memory()
o = torch.empty_like(x).pin_memory()
p = dwt2.Plan(16384, 16384, 1)
p.forward_host(x, o)
t = time.perf_counter()
for _ in range(5):
    p.forward_host(x, o)
dt = (time.perf_counter() - t) / 5
print(f"forward_host c3: {dt * 1e3:.2f} ms/step = {n / dt / 1e9:.2f} Gpix/s")
