"""Tile timeline of one pyramid launch (a -DDWT2_PROF build via DWT2_LIB, with
DWT2_PYRAMID=1): per level of the launch, tiles, first start, median start,
last end; and the number of tiles in progress over time."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
import _variant  # noqa: E402,F401
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
W, L = int(sys.argv[1]), int(sys.argv[2])
x = torch.from_numpy(workloads.smooth_noise(W, W, 4)).cuda()
y = torch.empty_like(x)
p = dwt2.Plan(W, W, L)
lib = dwt2.lib()
N = 1 << 16
buf = (ctypes.c_ulonglong * (3 * N))()
for it in range(3):
    p.forward(x, y)
torch.cuda.synchronize()
lib.dwt2_debug_tiles(buf, N)
a = np.frombuffer(buf, dtype=np.uint64).reshape(N, 3)
idx = np.nonzero(a[:, 1] != 0)[0]
used = a[:, 1] != 0
a = a[used]
st = (a[:, 0] >> 8).astype(np.int64)
lv = (a[:, 0] & 0xff).astype(np.int64)
en = (a[:, 1] >> 8).astype(np.int64)
t0 = st.min()
st, en = (st - t0) / 1e3, (en - t0) / 1e3
print(os.environ.get("TAG", ""), f"{W}^2 L{L}: {used.sum()} tiles, span {en.max():.1f} us")
for k in range(lv.max() + 1):
    s = lv == k
    if s.any():
        d = en[s] - st[s]
        print(f"  level {k}: {s.sum():6d} tiles  start {st[s].min():6.1f} / med {np.median(st[s]):6.1f} / max {st[s].max():6.1f}"
              f"  end max {en[s].max():6.1f}  tile dur med {np.median(d):5.2f} p90 {np.percentile(d, 90):5.2f}")
bins = np.arange(0, en.max() + 2, 2.0)
act = [((st <= b) & (en > b)).sum() for b in bins]
print("  tiles in progress every 2 us:", " ".join(str(v) for v in act))
fe = (a[:, 2].astype(np.int64) - t0) / 1e3
sm = (a[:, 1] & 0xff).astype(np.int64)
np.savez(os.environ.get("OUT", "/tmp/tiles.npz"), idx=idx, st=st, en=en, fe=fe, lv=lv, sm=sm)
late = np.argsort(-st)[:12]
for i in late:
    print(f"  late tile {idx[i]} level {lv[i]} sm {sm[i]} fetched {fe[i]:.1f} start {st[i]:.1f} end {en[i]:.1f}")
