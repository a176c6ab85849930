"""Small calls of every kernel family, for compute-sanitizer (memcheck /
racecheck / synccheck / initcheck): forward (TMA and bulk-copy loaders,
vector and scalar stores, batched, multi-level), strips (interior + boundary,
multi-level), inverse (ring and LDG kernels), the five comparison schemes and
the K = 2 kernel (9/7).  Exits 0 if every result matches the single-image
forward (or the oracle-free invariants checked here)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1708_07853_b200 import distributed as D  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
ok = True
for (W, H, L) in [(300, 212, 3), (257, 130, 2), (1024, 96, 2), (64, 64, 4)]:
    x = torch.from_numpy(workloads.uniform_int(W, H, W + H)).cuda()
    p = dwt2.Plan(W, H, L)
    y = p.forward(x)
    r = p.inverse(y)
    if L <= 2:
        ok &= bool(torch.equal(r, x))
    for s in ["nonsep_naive", "nonsep_lifting", "nonsep_adapted", "sep_conv", "sep_lifting"]:
        if L <= 2:
            ok &= bool(torch.equal(p.forward_scheme(s, x), y))
        else:
            p.forward_scheme(s, x)
    p.close()
    for wv in ("cdf97", "cdf53_k2"):
        q = dwt2.Plan(W, H, L, wavelet=wv)
        z = q.forward(x)
        if wv == "cdf53_k2":
            ok &= bool(torch.equal(z, y))
        q.close()
# batched
xs = torch.from_numpy(np.stack([workloads.uniform_int(130, 70, i) for i in range(3)])).cuda()
pb = dwt2.Plan(130, 70, 2, max_count=3)
yb = pb.forward(xs)
ok &= bool(torch.equal(pb.inverse(yb), xs))
pb.close()
# strips: 3 ranks on one GPU, 2 levels, ghost rows copied from the neighbours
W, H, G, L = 200, 96, 3, 2
img = torch.from_numpy(workloads.uniform_int(W, H, 77)).cuda()
pyrs = [D.StripPyramid(W, H, g, G, L, device="cuda") for g in range(G)]
plans = [dwt2.StripPlan(W, H, q.r0, q.r1, L) for q in pyrs]
for q in pyrs:
    q.owned(0).copy_(img[q.r0:q.r1])
for k in range(L):
    for g, q in enumerate(pyrs):
        w, h, rb, re, gt, gb = q.geom[k]
        if gt:
            o = pyrs[g - 1]
            q.level_buffer(k)[0:2].copy_(o.level_buffer(k)[o.geom[k][4] + (rb - 2 - o.geom[k][2]):o.geom[k][4] + (rb - o.geom[k][2])])
        if gb:
            o = pyrs[g + 1]
            q.level_buffer(k)[gt + (re - rb)].copy_(o.level_buffer(k)[o.geom[k][4] + (re - o.geom[k][2])])
    for q, pl in zip(pyrs, plans):
        ll = q.owned(k + 1) if k + 1 < L else None
        pl.forward_level(k, q.bufs[k], ll, q.out, dwt2.DWT2_STRIP_INTERIOR)
        pl.forward_level(k, q.bufs[k], ll, q.out, dwt2.DWT2_STRIP_BOUNDARY)
full = np.zeros((H, W), np.float32)
for q in pyrs:
    D.place_pyramid_output(full, q.out.cpu().numpy(), W, H, q.r0, q.r1, L)
ref = dwt2.Plan(W, H, L).forward(img).cpu().numpy()
ok &= bool(np.array_equal(full, ref))
torch.cuda.synchronize()
print("sanitize driver ok" if ok else "sanitize driver MISMATCH")
sys.exit(0 if ok else 1)
