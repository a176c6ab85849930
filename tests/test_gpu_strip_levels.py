"""Multi-level row strips on one GPU: every rank's
StripPyramid lives on cuda:0 and the per-level ghost-row exchange is
emulated by copying the neighbours' owned rows (the message pattern itself
is covered by the gloo tests).  The placed strip pyramids must equal the
single-GPU dwt2_forward bit for bit (fp64 register arithmetic: the result is
independent of the decomposition, Pin-10) and the oracle within tolerance.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import distributed as D
from paper_1708_07853_b200 import dwt2, workloads
from tests._parity import compare

pytestmark = pytest.mark.gpu


def emulate_exchange(pyrs, k):
    """Fill level k's ghost rows of every rank from its neighbours' owned rows."""
    for g, p in enumerate(pyrs):
        w, h, rb, re, gt, gb = p.geom[k]
        if gt:
            q = pyrs[g - 1]
            qrb, qgt = q.geom[k][2], q.geom[k][4]
            p.level_buffer(k)[0:2].copy_(q.level_buffer(k)[qgt + (rb - 2 - qrb):qgt + (rb - qrb)])
        if gb:
            q = pyrs[g + 1]
            qrb, qgt = q.geom[k][2], q.geom[k][4]
            p.level_buffer(k)[gt + (re - rb)].copy_(q.level_buffer(k)[qgt + (re - qrb)])


def run_strip_pyramids(x: np.ndarray, G: int, L: int, overlap: bool) -> np.ndarray:
    H, W = x.shape
    xt = torch.from_numpy(x).cuda()
    pyrs, plans = [], []
    for g in range(G):
        p = D.StripPyramid(W, H, g, G, L, device="cuda")
        p.owned(0).copy_(xt[p.r0:p.r1])
        pyrs.append(p)
        plans.append(dwt2.StripPlan(W, H, p.r0, p.r1, L))
    part_sets = ([dwt2.DWT2_STRIP_INTERIOR, dwt2.DWT2_STRIP_BOUNDARY] if overlap else [dwt2.DWT2_STRIP_ALL])
    for k in range(L):
        emulate_exchange(pyrs, k)
        for p, plan in zip(pyrs, plans):
            ll = p.owned(k + 1) if k + 1 < L else None
            for part in part_sets:
                plan.forward_level(k, p.bufs[k], ll, p.out, part)
    full = np.full((H, W), np.nan, np.float32)
    for p in pyrs:
        D.place_pyramid_output(full, p.out.cpu().numpy(), W, H, p.r0, p.r1, L)
    for plan in plans:
        plan.close()
    return full


@pytest.mark.parametrize("W,H,G,L", [
    (64, 64, 2, 3), (130, 97, 3, 2), (1000, 1030, 4, 4), (333, 2049, 8, 3), (4096, 4096, 8, 5),
    (1537, 1025, 3, 6), (257, 512, 2, 8)])
@pytest.mark.parametrize("overlap", [False, True])
def test_strip_pyramid_equals_single_gpu(W, H, G, L, overlap):
    x = workloads.uniform_real(W, H, W + 11 * H + L)
    got = run_strip_pyramids(x, G, L, overlap)
    plan = dwt2.Plan(W, H, L)
    ref = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    plan.close()
    assert not np.isnan(got).any()
    np.testing.assert_array_equal(got, ref)
    x64 = x.astype(np.float64)
    compare(got, oracle.forward(x64, L), oracle.forward(x64, L, round_f32=True), False, f"strips {W}x{H} G{G} L{L}")


def test_config4_on_8_strips_bit_identical():
    """Config 4 (8192^2 smooth + noise, 8 levels) split into 8 strips with one
    exchange per level: bit-identical to the single-GPU pyramid; and the odd
    8193^2 companion likewise."""
    for W in (8192, 8193):
        x = workloads.smooth_noise(W, W, 4)
        got = run_strip_pyramids(x, 8, 8, True)
        plan = dwt2.Plan(W, W, 8)
        ref = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        plan.close()
        np.testing.assert_array_equal(got, ref)


def test_strip_level_info_matches_python_geometry():
    for W, H, G, L in [(100, 1030, 4, 4), (33, 97, 3, 2), (8193, 8193, 8, 8)]:
        for g in range(G):
            r0, r1 = D.strip_rows_levels(H, g, G, L)
            plan = dwt2.StripPlan(W, H, r0, r1, L)
            py = D.level_rows(W, H, r0, r1, L)
            for k, info in enumerate(plan.level_info):
                assert (info.width, info.global_height, info.row_begin, info.row_end, info.ghost_top,
                        info.ghost_bot) == py[k]
            plan.close()


def test_strip_levels_rejects_misaligned():
    with pytest.raises(dwt2.DWT2Error):
        dwt2.StripPlan(64, 256, 4, 128, 3)        # row_begin not a multiple of 8
    with pytest.raises(dwt2.DWT2Error):
        dwt2.StripPlan(64, 256, 0, 100, 3)        # row_end not a multiple of 8 and not H
    with pytest.raises(dwt2.DWT2Error):
        dwt2.StripPlan(64, 257, 256, 257, 8)      # a 1-row strip


@pytest.mark.parametrize("overlap", [True, False])
def test_strip_pyramid_step_config3_g8(overlap):
    """The bench's per-rank step (strip_pyramid_step: the interior launch,
    the exchange's wait, then the boundary launch, all on the current stream)
    for every rank of config 3 at G = 8, with the exchange emulated by copying
    the ghost rows from the full image: bit-identical to the single-GPU
    transform."""
    x = workloads.uniform_int(16384, 16384, 3)
    H, W = x.shape
    xt = torch.from_numpy(x).cuda()
    full = np.full((H, W), np.nan, np.float32)
    for g in range(8):
        p = D.StripPyramid(W, H, g, 8, 1, device="cuda")
        p.owned(0).copy_(xt[p.r0:p.r1])
        plan = dwt2.StripPlan(W, H, p.r0, p.r1, 1)

        def exchange(k, p=p):
            lo, hi = p.global_rows(0)
            if p.ghost_top:
                p.bufs[0][0:2].copy_(xt[lo:lo + 2])
            if p.ghost_bot:
                p.bufs[0][-1].copy_(xt[hi - 1])
            return []
        D.strip_pyramid_step(p, plan, overlap=overlap, exchange=exchange)
        torch.cuda.synchronize()
        D.place_pyramid_output(full, p.out.cpu().numpy(), W, H, p.r0, p.r1, 1)
        plan.close()
    ref = dwt2.Plan(W, H, 1).forward(xt).cpu().numpy()
    np.testing.assert_array_equal(full, ref)


# ---------------------------------------------------------------------------
# The overlap contract of the real exchange, emulated asynchronously: the ghost
# rows are poisoned with NaN, and their copy runs on a second stream behind a
# ~1 ms spin kernel, so it lands while (or after) the INTERIOR launch runs; the
# BOUNDARY launch is ordered after it by current_stream().wait_event(), which is
# what NCCL's Work.wait() does.  An INTERIOR launch that read a ghost row, or a
# BOUNDARY launch that ran before the wait, would pick up a NaN.
# ---------------------------------------------------------------------------
SPIN_CYCLES = 2_000_000          # ~1 ms at 1.9 GHz


class _EventWait:
    def __init__(self, ev):
        self.ev = ev

    def wait(self):
        torch.cuda.current_stream().wait_event(self.ev)


def _poison_ghosts(p, k):
    w, h, rb, re, gt, gb = p.geom[k]
    buf = p.level_buffer(k)
    if gt:
        buf[0:gt].fill_(float("nan"))
    if gb:
        buf[gt + (re - rb):].fill_(float("nan"))


def run_strip_pyramids_async(x: np.ndarray, G: int, L: int) -> np.ndarray:
    H, W = x.shape
    xt = torch.from_numpy(x).cuda()
    cur = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    pyrs, plans = [], []
    for g in range(G):
        p = D.StripPyramid(W, H, g, G, L, device="cuda")
        p.owned(0).copy_(xt[p.r0:p.r1])
        pyrs.append(p)
        plans.append(dwt2.StripPlan(W, H, p.r0, p.r1, L))
    for k in range(L):
        for p in pyrs:
            _poison_ghosts(p, k)
        ready = torch.cuda.Event()
        ready.record(cur)                 # level k-1 of every rank done, ghosts poisoned
        with torch.cuda.stream(side):
            side.wait_event(ready)
            torch.cuda._sleep(SPIN_CYCLES)
            emulate_exchange(pyrs, k)     # the "receives"
            landed = torch.cuda.Event()
            landed.record(side)
        req = _EventWait(landed)
        for p, plan in zip(pyrs, plans):
            ll = p.owned(k + 1) if k + 1 < L else None
            plan.forward_level(k, p.bufs[k], ll, p.out, dwt2.DWT2_STRIP_INTERIOR)
        assert not landed.query(), "the emulated exchange finished before the interior launches were queued"
        req.wait()
        for p, plan in zip(pyrs, plans):
            ll = p.owned(k + 1) if k + 1 < L else None
            plan.forward_level(k, p.bufs[k], ll, p.out, dwt2.DWT2_STRIP_BOUNDARY)
    full = np.full((H, W), np.nan, np.float32)
    for p in pyrs:
        D.place_pyramid_output(full, p.out.cpu().numpy(), W, H, p.r0, p.r1, L)
    for plan in plans:
        plan.close()
    return full


@pytest.mark.parametrize("W,H,G,L", [(64, 64, 2, 3), (1000, 1030, 4, 4), (333, 2049, 8, 3), (4096, 4096, 8, 5),
                                     (8192, 8192, 8, 8), (8193, 8193, 8, 8)])
def test_strip_exchange_in_flight_during_interior(W, H, G, L):
    x = workloads.smooth_noise(W, H, 4) if W >= 8192 else workloads.uniform_real(W, H, W + 5 * H + L)
    got = run_strip_pyramids_async(x, G, L)
    plan = dwt2.Plan(W, H, L)
    ref = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    plan.close()
    assert not np.isnan(got).any()
    np.testing.assert_array_equal(got, ref)


def test_strip_pyramid_step_async_exchange_config3_g8():
    """strip_pyramid_step itself with an asynchronous exchange (poisoned ghost
    rows filled on a side stream behind a spin kernel, request.wait() =
    current_stream().wait_event()) on every rank of config 3 at G = 8."""
    x = workloads.uniform_int(16384, 16384, 3)
    H, W = x.shape
    xt = torch.from_numpy(x).cuda()
    cur = torch.cuda.current_stream()
    side = torch.cuda.Stream()
    full = np.full((H, W), np.nan, np.float32)
    for g in range(8):
        p = D.StripPyramid(W, H, g, 8, 1, device="cuda")
        p.owned(0).copy_(xt[p.r0:p.r1])
        plan = dwt2.StripPlan(W, H, p.r0, p.r1, 1)

        def exchange(k, p=p):
            _poison_ghosts(p, 0)
            ready = torch.cuda.Event()
            ready.record(cur)
            lo, hi = p.global_rows(0)
            with torch.cuda.stream(side):
                side.wait_event(ready)
                torch.cuda._sleep(SPIN_CYCLES)
                if p.ghost_top:
                    p.bufs[0][0:2].copy_(xt[lo:lo + 2])
                if p.ghost_bot:
                    p.bufs[0][-1].copy_(xt[hi - 1])
                landed = torch.cuda.Event()
                landed.record(side)
            return [_EventWait(landed)]
        D.strip_pyramid_step(p, plan, overlap=True, exchange=exchange)
        torch.cuda.synchronize()
        D.place_pyramid_output(full, p.out.cpu().numpy(), W, H, p.r0, p.r1, 1)
        plan.close()
    ref = dwt2.Plan(W, H, 1).forward(xt).cpu().numpy()
    np.testing.assert_array_equal(full, ref)
