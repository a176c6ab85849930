"""Buffer-pair count sensitivity per loader: config 2's shape (4096^2, 1
level), K = 20 graph-captured calls cycling over P pairs, for the 5/3
forward (TMA tensor loads), the 5/3 inverse (cp.async / LSU loads), the
K = 2 (9/7) forward (cp.async) and a device copy."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
W = H = 4096
x = torch.from_numpy(workloads.GENERATORS["smooth"](W, H, 2)).cuda()
p = dwt2.Plan(W, H, 1)
p97 = dwt2.Plan(W, H, 1, wavelet="cdf97")
y = p.forward(x).clone()
for P in (1, 3, 4, 8, 20):
    pf = [(x.clone(), torch.empty_like(x)) for _ in range(P)]
    pi = [(y.clone(), torch.empty_like(x)) for _ in range(P)]
    a = time_calls(lambda q: p.forward(q[0], q[1]), pf, 20)
    b = time_calls(lambda q: p.inverse(q[0], q[1]), pi, 20)
    c = time_calls(lambda q: p97.forward(q[0], q[1]), pf, 20)
    d = time_calls(lambda q: q[1].copy_(q[0]), pf, 20)
    print(f"P {P:2d}: forward 5/3 (TMA) {a:5.1f} | inverse 5/3 (cp.async) {b:5.1f} | forward 9/7 (cp.async) {c:5.1f} | "
          f"copy {d:5.1f} us", flush=True)
    del pf, pi
