"""The copy roofline at the bench's sizes: torch's device-to-device copy of a
W x H fp32 image (read 4 + write 4 bytes per pixel, as one DWT level), K
graph-captured calls on K distinct buffer pairs when the pair fits twice in
L2 (the bench's protocol).  Fraction of the large-copy peak of
MEASURED_PEAKS.json (6535 GB/s) -- what a level kernel of that size could
reach at best."""
import sys

import torch

sys.path.insert(0, "scripts")
from _timing import n_pairs, time_calls  # noqa: E402

torch.cuda.set_device(0)
K = 20
for W, H in [(512, 512), (2048, 2048), (4096, 4096), (8192, 8192), (16384, 2048), (16384, 16384)]:
    np_ = n_pairs(8 * W * H, K)
    pairs = [(torch.rand(H, W, device="cuda"), torch.empty(H, W, device="cuda")) for _ in range(np_)]
    us = time_calls(lambda q: q[1].copy_(q[0]), pairs, K)
    gbs = 8.0 * W * H / us / 1e3
    print(f"copy {W}x{H}: {us:8.1f} us  {gbs:6.0f} GB/s  ({gbs / 6535:.3f} of the large-copy peak)")
    del pairs
