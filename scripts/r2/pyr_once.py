"""One forward of a config-5-like group (n x W^2, L levels) for ncu captures."""
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import _variant  # noqa: E402,F401
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

W, L, n = (int(v) for v in sys.argv[1:4])
x = torch.from_numpy(workloads.uniform_int(W, W * n, 5).reshape(n, W, W)).cuda()
y = torch.empty_like(x)
p = dwt2.Plan(W, W, L, max_count=n)
for _ in range(3):
    p.forward(x, y)
torch.cuda.synchronize()
