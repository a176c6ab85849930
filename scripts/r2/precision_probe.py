"""fp64 vs fp32 register arithmetic: max-abs error against the
fp64 oracle (i) of the library given by DWT2_LIB (product: fp64 registers;
-DDWT2_F32MATH / -DDWT2_K2_F32 builds: fp32 registers) on configs 2, 4 and 4b
(CDF 5/3) and on the config-4 shape with CDF 9/7, over 4 seeds each, plus the
mismatch count against oracle (ii)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import _variant  # noqa: E402,F401
import oracle  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
tag = os.environ.get("TAG", "")
cases = [("c2", 4096, 4096, 1, "cdf53"), ("c4", 8192, 8192, 8, "cdf53"), ("c4b", 8193, 8193, 8, "cdf53"),
         ("c4-97", 8192, 8192, 8, "cdf97")]
only = os.environ.get("CASES")
for name, W, H, L, wav in cases:
    if only and name not in only.split(","):
        continue
    worst_i, worst_ii, nbad = 0.0, 0.0, 0
    for seed in range(4):
        x = workloads.smooth_noise(W, H, 40 + seed)
        plan = dwt2.Plan(W, H, L, wavelet=wav)
        y = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
        plan.close()
        x64 = x.astype(np.float64)
        ref_i = oracle.forward(x64, L, round_f32=False, wavelet=wav)
        worst_i = max(worst_i, float(np.abs(y - ref_i).max()))
        ref_ii = oracle.forward(x64, L, round_f32=True, wavelet=wav)
        d = np.abs(y - ref_ii)
        worst_ii = max(worst_ii, float(d.max()))
        nbad += int(np.count_nonzero(d))
    print(f"{tag} {name} ({wav}, {W}x{H}, L{L}, 4 seeds): max|gpu - oracle(i)| = {worst_i:.3e}, "
          f"max|gpu - oracle(ii)| = {worst_ii:.3e}, elements != oracle(ii): {nbad}", flush=True)
