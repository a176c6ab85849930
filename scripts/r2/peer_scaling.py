"""Row strips on one GPU, all G ranks of a step emulated in one stream: the
peer-memory halo path (DWT2_PEER_SEQUENTIAL: per level every rank's INTERIOR
launch, then every rank's BOUNDARY launch with its peer reads) against the
NCCL path with the exchange stubbed (strip_pyramid_step, no copy), both as
K steps in one CUDA graph.  Sum over the G ranks per step; divided by G it is
the mean per-rank GPU time of a step, and T(1) / sum the strong-scaling
efficiency the step's GPU work allows with perfect overlap of the ranks."""
import sys
import time

import torch

sys.path.insert(0, ".")
sys.path.insert(0, "scripts")
from _timing import time_calls  # noqa: E402
from paper_1708_07853_b200 import distributed as D  # noqa: E402
from paper_1708_07853_b200 import dwt2, workloads  # noqa: E402

torch.cuda.set_device(0)
noop = lambda k: []  # noqa: E731
for name, W, H, L in [("config 3", 16384, 16384, 1), ("config 4", 8192, 8192, 8), ("config 2", 4096, 4096, 1)]:
    x = torch.from_numpy(workloads.uniform_int(W, H, 1)).cuda()
    y = torch.empty_like(x)
    p = dwt2.Plan(W, H, L)
    t1 = time_calls(lambda q: p.forward(q[0], q[1]), [(x, y)], 10)
    p.close()
    print(f"{name}: G=1 {t1:7.1f} us/step", flush=True)
    for G in (2, 4, 8):
        ranks = [D.PeerStripPyramid(W, H, g, G, L, device="cuda") for g in range(G)]
        for r in ranks:
            r.connect_local(ranks)
            r.strip.copy_(x[r.r0:r.r1])
        t_peer = time_calls(lambda q: D.sequential_step(ranks), [(None,)], 10)
        t_split = time_calls(lambda q: D.sequential_step(ranks, fused=False), [(None,)], 10)

        def publish_only(q):               # the emulation's PUBLISH launches alone (a rank on its own GPU has none)
            for k in range(L):
                for r in ranks:
                    r.ctx.level(k, dwt2.DWT2_STRIP_PUBLISH, r.out)
        t_pub = time_calls(publish_only, [(None,)], 10)
        torch.cuda.synchronize()
        h0 = time.perf_counter()
        for _ in range(20):
            D.sequential_step(ranks)
        h1 = time.perf_counter()
        torch.cuda.synchronize()
        st = [r.status() for r in ranks]
        for r in ranks:
            r.close()
        del ranks
        pyrs, plans = [], []
        for g in range(G):
            pyr = D.StripPyramid(W, H, g, G, L, device="cuda")
            pyr.strip.copy_(x[pyr.r0:pyr.r1])
            pyrs.append(pyr)
            plans.append(dwt2.StripPlan(W, H, pyr.r0, pyr.r1, L))

        def stub_step(q):
            for pyr, plan in zip(pyrs, plans):
                D.strip_pyramid_step(pyr, plan, overlap=True, exchange=noop)
        t_stub = time_calls(stub_step, [(None,)], 10)
        for plan in plans:
            plan.close()
        del pyrs
        print(f"{name}: G={G} peer fused {t_peer:7.1f} us / step of all ranks ({t_peer / G:6.1f} per rank, "
              f"{(t_peer - t_pub) / G:6.1f} without the emulation's {G * L} PUBLISH launches [{t_pub:5.1f} us], "
              f"T1/sum {t1 / t_peer:.2f}); peer split {t_split:7.1f} ({t_split / G:6.1f} per rank); "
              f"host enqueue {(h1 - h0) / 20 * 1e6 / G:5.1f} us per rank-step; "
              f"nccl-stub {t_stub:7.1f} us ({t_stub / G:6.1f} per rank, T1/sum {t1 / t_stub:.2f}); status {set(st)}",
              flush=True)
