"""Forward of a W x H image (for ncu captures): python scripts/one_level.py W H [reps] [levels]."""
import sys

import torch

sys.path.insert(0, ".")
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

W, H = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
levels = int(sys.argv[4]) if len(sys.argv) > 4 else 1
x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
p = dwt2.Plan(W, H, levels)
y = torch.empty_like(x)
for _ in range(reps):
    p.forward(x, y)
torch.cuda.synchronize()
print("ok", W, H)
