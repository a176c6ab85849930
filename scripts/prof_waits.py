"""Fraction of warp time spent waiting for TMA stages (needs a -DDWT2_PROF build via DWT2_LIB)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, '.')
sys.path.insert(0, "scripts")
import _variant  # noqa: E402,F401
from paper_1708_07853_b200 import dwt2, workloads
W = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
H = int(sys.argv[2]) if len(sys.argv) > 2 else W
x = torch.from_numpy(workloads.uniform_int(W, H, 3)).cuda()
out = torch.empty_like(x)
p = dwt2.Plan(W, H, 1)
lib = dwt2.lib()
buf = (ctypes.c_ulonglong * 4)()
for _ in range(3): p.forward(x, out)
torch.cuda.synchronize()
lib.dwt2_debug_prof(buf, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): p.forward(x, out)
e1.record(); torch.cuda.synchronize()
lib.dwt2_debug_prof(buf, 1)
wait, seg, stages = buf[0], buf[1], buf[2]
print(f"{W*H*10/e0.elapsed_time(e1)/1e6:.1f} Gpix/s  wait/segment cycles = {wait/seg:.3f}  cycles per stage (per warp) = {seg/max(stages,1):.0f}  wait per stage = {wait/max(stages,1):.0f}")
# per-CTA timeline of the last launch
n = 4096
arr = (ctypes.c_ulonglong * (4 * n))()
p.forward(x, out); torch.cuda.synchronize()
lib.dwt2_debug_cta(arr, n)
a = np.frombuffer(arr, dtype=np.uint64).reshape(n, 4).astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
ent, s0, s1 = (a[:, 0] - t0) / 1e3, (a[:, 1] - t0) / 1e3, (a[:, 2] - t0) / 1e3
print(f"CTAs {len(a)}  entry us: min {ent.min():.1f} med {np.median(ent):.1f} max {ent.max():.1f}; work start med {np.median(s0):.1f}; end min {s1.min():.1f} med {np.median(s1):.1f} max {s1.max():.1f}")
sm = a[:, 3]
cnt = np.bincount(sm, minlength=148)
print("CTAs per SM histogram:", np.bincount(cnt))
dur = s1 - s0
for c in sorted(set(cnt)):
    sel = np.isin(sm, np.where(cnt == c)[0])
    if sel.any(): print(f"  SMs with {c} CTAs: seg duration med {np.median(dur[sel]):.1f} us max {dur[sel].max():.1f}")
