"""Multi-process host logic of the multi-GPU paths, on CPU with the gloo backend.

* Row strips (config 3): after StripExchange's grouped send/recv, every
  rank's input buffer must equal the global image rows
  [r_g - ghost_top, r_{g+1} + ghost_bot) -- exactly what the level kernel
  reads (2 ghost rows above, 1 below; Eq. (5) supports).  Strip
  outputs placed by place_strip_output must tile the global Mallat layout.
* Batches (config 5): shards cover every image exactly once.

world sizes 2 and 3 (an interior rank has both neighbours).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1708_07853_b200 import distributed as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, W, H, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = (np.arange(H * W, dtype=np.float32).reshape(H, W) % 251.0).astype(np.float32)
        ex = D.StripExchange(W, H, rank, world, device="cpu")
        ex.buf.fill_(-1.0)
        ex.strip.copy_(torch.from_numpy(img[ex.r0:ex.r1]))
        reqs = ex.start()
        ex.finish(reqs)
        lo, hi = ex.r0 - ex.ghost_top, ex.r1 + ex.ghost_bot
        ok = np.array_equal(ex.buf.numpy(), img[lo:hi])
        q.put((rank, ok, ex.r0, ex.r1, ex.ghost_top, ex.ghost_bot))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H", [(2, 40, 30), (3, 33, 17), (3, 64, 64)])
def test_strip_halo_exchange_gloo(world, W, H):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, W, H, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    for rank, ok, r0, r1, gt, gb in res:
        assert ok, f"rank {rank}: ghost rows wrong"
        assert gt == (2 if r0 > 0 else 0) and gb == (1 if r1 < H else 0)
    # strips tile the image
    assert res[0][2] == 0 and res[-1][3] == H
    for a, b in zip(res, res[1:]):
        assert a[3] == b[2] and a[2] % 2 == 0


def test_strip_partition_rules():
    for H in [2, 3, 17, 64, 101, 16384]:
        for G in [1, 2, 3, 4, 8]:
            if H < 2 * G:
                continue
            prev = 0
            for g in range(G):
                r0, r1 = D.strip_rows(H, g, G)
                assert r0 == prev and r0 % 2 == 0 and r1 > r0
                assert (r1 % 2 == 0) or r1 == H
                prev = r1
            assert prev == H
            sizes = [D.strip_rows(H, g, G)[1] - D.strip_rows(H, g, G)[0] for g in range(G)]
            assert max(sizes) - min(sizes) <= 3


def test_halo_plan_messages_match():
    """Every send has a matching receive on the peer with the same row count."""
    H, G = 100, 4
    plans = {g: D.halo_plan(H, g, G) for g in range(G)}
    for g, msgs in plans.items():
        for op, peer, _, n in msgs:
            if op == "send":
                assert ("recv", g, n) in [(o, p, m) for o, p, _, m in plans[peer]]


def test_place_and_take_strip_output_roundtrip():
    rng = np.random.default_rng(0)
    for W, H, G in [(10, 14, 3), (9, 17, 4), (16, 16, 2)]:
        full = rng.standard_normal((H, W)).astype(np.float32)
        rebuilt = np.full_like(full, np.nan)
        for g in range(G):
            r0, r1 = D.strip_rows(H, g, G)
            D.place_strip_output(rebuilt, D.take_strip_output(full, W, H, r0, r1), W, H, r0, r1)
        np.testing.assert_array_equal(rebuilt, full)


def test_batch_shards_cover():
    for count in [1, 5, 32, 256]:
        for G in [1, 2, 3, 8]:
            seen = []
            for g in range(G):
                seen.extend(D.shard(count, g, G))
            assert seen == list(range(count))


# --------------------------------------------------------------------------
# multi-level strips: one exchange per level
# --------------------------------------------------------------------------

def _level_image(W, H, k):
    """Synthetic stand-in for level k's input (the exchange moves rows; their
    values do not matter, only that every ghost row is the right global row)."""
    return ((np.arange(H * W, dtype=np.float64).reshape(H, W) * (k + 3)) % 997.0).astype(np.float32)


def _worker_levels(rank, world, port, W, H, L, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pyr = D.StripPyramid(W, H, rank, world, L, device="cpu")
        oks = []
        for k, (w, h, rb, re, gt, gb) in enumerate(pyr.geom):
            img = _level_image(w, h, k)
            pyr.bufs[k].fill_(-1.0)
            pyr.owned(k).copy_(torch.from_numpy(img[rb:re]))
            pyr.finish(pyr.start(k))
            lo, hi = pyr.global_rows(k)
            oks.append(bool(np.array_equal(pyr.level_buffer(k).numpy(), img[lo:hi])))
        q.put((rank, oks, pyr.r0, pyr.r1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H,L", [(2, 40, 64, 3), (3, 33, 97, 2), (3, 20, 130, 4)])
def test_multilevel_strip_exchange_gloo(world, W, H, L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_levels, args=(r, world, port, W, H, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, oks, r0, r1 in res:
        assert all(oks), f"rank {rank}: ghost rows wrong at levels {[k for k, o in enumerate(oks) if not o]}"
    assert res[0][2] == 0 and res[-1][3] == H
    for a, b in zip(res, res[1:]):
        assert a[3] == b[2] and a[3] % (1 << L) == 0


def test_multilevel_partition_and_geometry():
    for H in [64, 97, 130, 8193, 16384]:
        for G in [1, 2, 3, 8]:
            for L in [1, 2, 3, 8]:
                unit = 1 << L
                if -(-H // unit) < G:
                    continue
                prev = 0
                for g in range(G):
                    r0, r1 = D.strip_rows_levels(H, g, G, L)
                    assert r0 == prev and r0 % unit == 0 and (r1 % unit == 0 or r1 == H)
                    prev = r1
                    geom = D.level_rows(64, H, r0, r1, L)
                    # each level's strips tile that level's image
                    for k, (w, h, rb, re, gt, gb) in enumerate(geom):
                        assert rb == r0 >> k and rb % 2 == 0
                        assert gt == (2 if rb else 0) and gb == (1 if re < h else 0)
                assert prev == H


def test_place_pyramid_output_tiles_global():
    """Strip-local pyramids placed per rank rebuild the global Mallat pyramid
    (every element written exactly once) -- checked on index maps."""
    for W, H, G, L in [(24, 64, 2, 3), (17, 97, 3, 2), (40, 130, 3, 4)]:
        cover = np.zeros((H, W), np.int32)
        for g in range(G):
            r0, r1 = D.strip_rows_levels(H, g, G, L)
            mark = np.zeros((H, W), np.int32)
            D.place_pyramid_output(mark, np.ones((r1 - r0, W), np.int32), W, H, r0, r1, L)
            cover += mark
        assert (cover == 1).all(), np.argwhere(cover != 1)[:5]


# --------------------------------------------------------------------------
# the per-rank step of the bench (strip_pyramid_step) over gloo, with the
# level kernels replaced by a host stand-in that checks what the real kernel
# relies on: at every BOUNDARY launch the ghost rows hold the neighbours'
# rows of that level's image, and the launch arguments are the level's
# buffers.  The stand-in "produces" level k+1's owned rows (a known function
# of the global row), so the next level's exchange moves data written by
# the previous level's launches -- the cross-rank ordering of the step.
# --------------------------------------------------------------------------

def _level_value(k, rows, w):
    """Synthetic content of level k's input, global rows `rows` (array), w columns."""
    return ((rows[:, None] * 7 + np.arange(w)[None, :] * 3 + k * 101) % 1009).astype(np.float32)


class _FakeStripPlan:
    def __init__(self, pyr):
        self.pyr, self.handle, self.calls = pyr, 12345, []

    def launch_level(self, h, k, bp, bpitch, lp, lpitch, out, part, stream):
        pyr = self.pyr
        w, hgt, rb, re, gt, gb = pyr.geom[k]
        assert h == 12345 and bp == pyr.bufs[k].data_ptr() and bpitch == pyr.bufs[k].stride(0)
        if k + 1 < pyr.levels:
            assert lp == pyr.owned(k + 1).data_ptr() and lpitch == pyr.owned(k + 1).stride(0)
        if part == 2:       # BOUNDARY: ghost rows must be the neighbours' rows of this level
            lo, hi = pyr.global_rows(k)
            exp = _level_value(k, np.arange(lo, hi), w)
            got = pyr.level_buffer(k).numpy()
            assert np.array_equal(got[:gt], exp[:gt]) and np.array_equal(got[got.shape[0] - gb:], exp[exp.shape[0] - gb:])
        self.calls.append((k, part))
        if k + 1 < pyr.levels:      # "write" level k+1's owned rows (interior: all but first/last, boundary: those)
            w1, h1, rb1, re1, _, _ = pyr.geom[k + 1]
            own = pyr.owned(k + 1).numpy()
            vals = _level_value(k + 1, np.arange(rb1, re1), w1)
            sel = np.zeros(re1 - rb1, bool)
            if part == 1:
                sel[1:-1] = True
            elif part == 2:
                sel[0] = sel[-1] = True
            else:
                sel[:] = True
            own[sel] = vals[sel]


def _worker_step(rank, world, port, W, H, L, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        pyr = D.StripPyramid(W, H, rank, world, L, device="cpu")
        w0, h0, rb0, re0, _, _ = pyr.geom[0]
        pyr.owned(0).copy_(torch.from_numpy(_level_value(0, np.arange(rb0, re0), w0)))
        plan = _FakeStripPlan(pyr)
        for _ in range(2):                      # two steps: the exchange state is reusable
            D.strip_pyramid_step(pyr, plan, overlap=True)
        q.put((rank, plan.calls))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H,L", [(2, 48, 64, 3), (3, 30, 130, 2)])
def test_strip_pyramid_step_gloo(world, W, H, L):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_step, args=(r, world, port, W, H, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, calls in res:
        assert calls == [(k, part) for _ in range(2) for k in range(L) for part in (1, 2)]


# ---- peer-memory halo: descriptor exchange (the GPU side is test_gpu_peer_strips.py)

def _fake_desc(W, H, rank, world, L):
    """The geometry fields dwt2_peer_strip_export fills (no GPU here)."""
    from paper_1708_07853_b200 import dwt2
    d = dwt2.PeerDesc()
    d.width, d.global_height, d.levels = W, H, L
    d.row_begin, d.row_end = D.strip_rows_levels(H, rank, world, L)
    d.pid, d.device, d.base = os.getpid(), rank, 0x7f0000000000 + rank * (1 << 30)
    for k, (w, h, rb, re, gt, gb) in enumerate(D.level_rows(W, H, d.row_begin, d.row_end, L)):
        d.pitch[k] = -(-w // 4) * 4
        d.owned_off[k] = 4096 * k + gt * 4 * d.pitch[k]
    return d


def _peer_worker(rank, world, port, W, H, L, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        descs = D.gather_descriptors(_fake_desc(W, H, rank, world, L).to_bytes())
        above, below = D.peer_neighbours(descs, rank)
        q.put((rank, None if above is None else (above.row_begin, above.row_end, above.pid, above.device),
               None if below is None else (below.row_begin, below.row_end, below.pid, below.device), os.getpid()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,W,H,L", [(2, 64, 64, 1), (3, 100, 1030, 4), (4, 33, 97, 2)])
def test_peer_descriptor_exchange_gloo(world, W, H, L):
    """Every rank gets the descriptor of the rank owning the rows just above
    (None for rank 0) and just below (None for the last rank), in the process
    that exported it (its pid and device travel with it)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_peer_worker, args=(r, world, port, W, H, L, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r: (a, b, pid) for r, a, b, pid in (q.get(timeout=120) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        a, b, _ = res[r]
        lo, hi = D.strip_rows_levels(H, r, world, L)
        if r == 0:
            assert a is None
        else:
            assert a == (*D.strip_rows_levels(H, r - 1, world, L), res[r - 1][2], r - 1) and a[1] == lo
        if r == world - 1:
            assert b is None
        else:
            assert b == (*D.strip_rows_levels(H, r + 1, world, L), res[r + 1][2], r + 1) and b[0] == hi


def test_peer_neighbours_rejects_mismatched_geometry():
    descs = [_fake_desc(64, 64, r, 3, 2).to_bytes() for r in range(3)]
    above, below = D.peer_neighbours(descs, 1)
    assert (above.row_end, below.row_begin) == D.strip_rows_levels(64, 1, 3, 2)
    bad = _fake_desc(64, 64, 2, 3, 2)
    bad.row_begin += 4                      # a gap between rank 1 and rank 2
    with pytest.raises(ValueError):
        D.peer_neighbours([descs[0], descs[1], bad.to_bytes()], 1)
    bad = _fake_desc(64, 64, 0, 3, 2)
    bad.levels = 3
    with pytest.raises(ValueError):
        D.peer_neighbours([bad.to_bytes(), descs[1], descs[2]], 1)
