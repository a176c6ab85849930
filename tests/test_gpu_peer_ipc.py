"""The peer strip path across PROCESSES: two ranks as two processes on
cuda:0, whose contexts map each other through CUDA IPC
(cudaIpcGetMemHandle / cudaIpcOpenMemHandle -- the mapping a rank on its own
GPU uses for its NVLink neighbour).  No kernel ever waits for the other
process: the host orders the phases with a barrier (per level: both ranks'
PUBLISH launches, then rank 0's fused launch, then rank 1's), so every flag a
launch acquires -- across the process boundary -- is already published, and
the boundary rows are read from the other process's allocation.  The placed
pyramid must be bit-exact against oracle (ii)."""
import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

import oracle
from paper_1708_07853_b200 import workloads

pytestmark = pytest.mark.gpu

W, H, G, L = 300, 256, 2, 3


def _rank(rank, q_desc, q_in, q_out, bar):
    import torch
    from paper_1708_07853_b200 import distributed as D
    from paper_1708_07853_b200 import dwt2
    torch.cuda.set_device(0)
    try:
        x = workloads.uniform_real(W, H, 11)
        r = D.PeerStripPyramid(W, H, rank, G, L, device="cuda")
        r.strip.copy_(torch.from_numpy(x[r.r0:r.r1]).cuda())
        torch.cuda.synchronize()
        q_desc.put((rank, r.export()))
        descs = q_in.get(timeout=120)
        r.connect_descriptors(descs, dwt2.DWT2_PEER_SEQUENTIAL)
        for step in range(2):
            for k in range(L):
                r.ctx.level(k, dwt2.DWT2_STRIP_PUBLISH, r.out)
                torch.cuda.synchronize()
                bar.wait(timeout=120)
                for turn in range(G):
                    if turn == rank:
                        r.ctx.level(k, dwt2.DWT2_STRIP_ALL, r.out)
                        torch.cuda.synchronize()
                    bar.wait(timeout=120)
        q_out.put((rank, r.r0, r.r1, r.out.cpu().numpy(), r.status()))
        bar.wait(timeout=120)          # the neighbour is done reading this rank's memory
        r.close()
    except Exception as e:            # report, do not hang the parent
        q_out.put((rank, None, None, repr(e), -99))


def test_peer_strips_across_processes_via_cuda_ipc():
    from paper_1708_07853_b200 import distributed as D
    ctx = mp.get_context("spawn")
    q_desc, q_out = ctx.Queue(), ctx.Queue()
    q_in = [ctx.Queue() for _ in range(G)]
    bar = ctx.Barrier(G)
    procs = [ctx.Process(target=_rank, args=(g, q_desc, q_in[g], q_out, bar)) for g in range(G)]
    for p in procs:
        p.start()
    descs = [None] * G
    for _ in range(G):
        g, d = q_desc.get(timeout=300)
        descs[g] = d
    for g in range(G):
        q_in[g].put(descs)
    res = [q_out.get(timeout=300) for _ in range(G)]
    for p in procs:
        p.join(timeout=120)
    full = np.full((H, W), np.nan, np.float32)
    for g, r0, r1, out, status in res:
        assert status == 0, f"rank {g}: {out}"
        D.place_pyramid_output(full, out, W, H, r0, r1, L)
    x = workloads.uniform_real(W, H, 11)
    ref = oracle.forward(x.astype(np.float64), L, round_f32=True).astype(np.float32)
    np.testing.assert_array_equal(full, ref)
