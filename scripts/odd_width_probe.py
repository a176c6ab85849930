"""Level-1 forward time vs image width around 8192 (H = 8192): 3-D TMA loader
(row pitch a multiple of 16 bytes) against the row-grouped TMA loader (other
widths; the bulk-copy loader with a DWT2_NO_GRP build), and vector against
scalar subband stores.  In the Mallat layout a
pitch that is not a multiple of 16 bytes always comes with scalar stores
(HL starts at column ceil(W/2)), so the probe variants built with
DWT2_FORCE_GENERIC / DWT2_FORCE_SCALAR (DWT2_LIB=...) separate the two."""
import os
import sys

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
sys.path.insert(0, "scripts")
import _variant  # noqa: E402,F401
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
H = 8192
tag = os.path.basename(os.environ.get("DWT2_LIB", "libdwt2.so"))
for W in (8192, 8196, 8194, 8193, 8195, 8200):
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, 1)
    us = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 20)
    gbs = 8.0 * W * H / us / 1e3
    G = 1 if W % 4 == 0 else (2 if W % 2 == 0 else 4)
    loader = "3-D TMA" if G == 1 else f"row-grouped TMA, G = {G}"
    print(f"{tag} W={W}: {us:7.1f} us  {gbs:6.0f} GB/s  (pitch {4 * W} B: {loader} loader unless DWT2_NO_GRP, "
          f"{'vector' if W % 4 == 0 else 'scalar'} stores unless forced)")
    p.close()
