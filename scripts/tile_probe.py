"""Level-1 time of W x H images under the tile policy's environment knobs
(DWT2_TPW, DWT2_MIN_TB, ...): python scripts/tile_probe.py W H [W H ...].
PROBE_OP=inverse times the inverse, PROBE_WAVELET=cdf97 the K = 2 kernels,
PROBE_COLD=1 gives every call its own buffers (forward only) as bench.py does."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import n_pairs, time_calls  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
a = [int(v) for v in sys.argv[1:]] or [16384, 8192]
out = []
for W, H in zip(a[0::2], a[1::2]):
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, 1, wavelet=os.environ.get("PROBE_WAVELET", "cdf53"))
    if os.environ.get("PROBE_OP") == "inverse":
        x = p.forward(x).clone()
        pairs = [(x, y)]
        if os.environ.get("PROBE_COLD"):
            pairs += [(x.clone(), torch.empty_like(y)) for _ in range(n_pairs(8 * W * H, 10) - 1)]
        us = time_calls(lambda q: p.inverse(q[0], q[1]), pairs, 10)
    else:
        pairs = [(x, y)]
        if os.environ.get("PROBE_COLD"):      # the bench's protocol (buffer pairs cycled, cold L2)
            pairs += [(x.clone(), torch.empty_like(y)) for _ in range(n_pairs(8 * W * H, 10) - 1)]
        us = time_calls(lambda q: p.forward(q[0], q[1]), pairs, 10)
    out.append(f"{W}x{H} {us:.1f} us ({8 * W * H / us / 1e3 / 6535:.3f})")
    p.close()
print(" | ".join(out))
