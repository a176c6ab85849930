"""Small driver for ncu captures of one kernel: runs `reps` calls of the
selected operation on a config's image (no timing; use under ncu with -k)."""
import argparse
import sys

import torch

sys.path.insert(0, ".")
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("op", choices=["forward", "inverse", "forward97", "scheme"])
ap.add_argument("--config", default="3")
ap.add_argument("--levels", type=int, default=0)
ap.add_argument("--scheme", default="sep_lifting")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = workloads.CONFIGS[a.config]
g = cfg.groups[0]
L = a.levels or cfg.levels
x = torch.from_numpy(g.image(0)).cuda()
plan = dwt2.Plan(g.width, g.height, L, wavelet="cdf97" if a.op == "forward97" else "cdf53")
y = plan.forward(x)
o = torch.empty_like(x)
for _ in range(a.reps):
    if a.op in ("forward", "forward97"):
        plan.forward(x, o)
    elif a.op == "inverse":
        plan.inverse(y, o)
    else:
        plan.forward_scheme(a.scheme, x, o)
torch.cuda.synchronize()
print("ok")
