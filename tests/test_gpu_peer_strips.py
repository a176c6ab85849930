"""Row strips with the halo read from peer memory inside the BOUNDARY kernel
(include/dwt2.h "peer strip context"; the exchange
point of PAPER.md L94-98).

Every rank's context lives on cuda:0 and the ranks run in ONE stream in the
DWT2_PEER_SEQUENTIAL order (per level: every rank's PUBLISH launch, then
every rank's fused launch; or every rank's INTERIOR launch, which publishes,
then every rank's BOUNDARY launch), so every flag a launch waits for was
published by an earlier launch.  Both level forms are covered: the fused one
(DWT2_STRIP_ALL: the level kernel plus boundary-role CTAs in ONE launch -- the
step's form) and the split one.  The placed strip pyramids must equal the single-GPU dwt2_forward bit
for bit and the oracle (ii) bit for bit (fp64 register arithmetic, the
per-level fp32 rounding of oracle (ii)).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import distributed as D
from paper_1708_07853_b200 import dwt2, workloads
from tests._parity import compare

pytestmark = pytest.mark.gpu


def make_ranks(W, H, G, L, timeout_ms=0):
    ranks = [D.PeerStripPyramid(W, H, g, G, L, device="cuda", timeout_ms=timeout_ms) for g in range(G)]
    for r in ranks:
        r.connect_local(ranks)
    return ranks


def fill(ranks, x):
    xt = torch.from_numpy(x).cuda()
    for r in ranks:
        r.strip.copy_(xt[r.r0:r.r1])


def gather(ranks, W, H, L):
    full = np.full((H, W), np.nan, np.float32)
    for r in ranks:
        D.place_pyramid_output(full, r.out.cpu().numpy(), W, H, r.r0, r.r1, L)
    return full


def single_gpu(x, L):
    H, W = x.shape
    plan = dwt2.Plan(W, H, L)
    ref = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    plan.close()
    return ref


def close(ranks):
    torch.cuda.synchronize()
    for r in ranks:
        assert r.status() == dwt2.DWT2_OK
        r.close()


@pytest.mark.parametrize("W,H,G,L", [
    (64, 64, 2, 1), (64, 64, 2, 3), (130, 97, 3, 2), (300, 212, 2, 1), (1000, 1030, 4, 4), (333, 2049, 8, 3),
    (4096, 4096, 8, 5), (1537, 1025, 3, 6), (257, 512, 2, 8), (8, 64, 4, 1), (5, 40, 5, 2), (1030, 16, 4, 2)])
@pytest.mark.parametrize("fused", [True, False])
def test_peer_strips_equal_single_gpu_and_oracle(W, H, G, L, fused):
    x = workloads.uniform_real(W, H, 3 * W + H + L)
    ranks = make_ranks(W, H, G, L)
    fill(ranks, x)
    D.sequential_step(ranks, fused=fused)
    got = gather(ranks, W, H, L)
    close(ranks)
    assert not np.isnan(got).any()
    np.testing.assert_array_equal(got, single_gpu(x, L))
    x64 = x.astype(np.float64)
    what = f"peer strips {W}x{H} G{G} L{L} fused={fused}"
    compare(got, None, oracle.forward(x64, L, round_f32=True), True, what)       # bit-exact vs oracle (ii)
    compare(got, oracle.forward(x64, L), None, False, what)                      # within 1e-4 of oracle (i)


def test_peer_strips_two_row_strips():
    """Strips of exactly 2 rows at the last level (the single boundary quad row
    reads 2 rows above AND 1 row below from the neighbours)."""
    for (W, H, G, L) in [(48, 32, 8, 1), (48, 16, 8, 1), (40, 64, 8, 2)]:
        x = workloads.uniform_int(W, H, W + H)
        for fused in (True, False):
            ranks = make_ranks(W, H, G, L)
            fill(ranks, x)
            D.sequential_step(ranks, fused=fused)
            got = gather(ranks, W, H, L)
            close(ranks)
            np.testing.assert_array_equal(got, oracle.forward(x.astype(np.float64), L, round_f32=True).astype(np.float32))


def test_peer_strips_config3_g8_and_config4_g8():
    """Config 3 (16384^2, 1 level) and config 4 (8192^2, 8 levels) on 8
    emulated ranks: bit-identical to the single-GPU transform."""
    for (W, L, x) in [(16384, 1, workloads.uniform_int(16384, 16384, 3)), (8192, 8, workloads.smooth_noise(8192, 8192, 4))]:
        ranks = make_ranks(W, W, 8, L)
        fill(ranks, x)
        D.sequential_step(ranks)
        got = gather(ranks, W, W, L)
        close(ranks)
        np.testing.assert_array_equal(got, single_gpu(x, L))
        del got


def test_peer_strips_repeated_steps_new_inputs():
    """Epochs advance on the device: several steps with new level-0 rows, each
    correct (stale rows or flags of an earlier step would show)."""
    W, H, G, L = 520, 384, 4, 3
    ranks = make_ranks(W, H, G, L)
    for s in range(6):
        x = workloads.uniform_real(W, H, 100 + s)
        fill(ranks, x)
        D.sequential_step(ranks, fused=s % 2 == 0)
        np.testing.assert_array_equal(gather(ranks, W, H, L), single_gpu(x, L))
    close(ranks)


def test_peer_strips_graph_capture():
    """The sequential step of all ranks captured in ONE CUDA graph and
    replayed with new inputs (no host work between levels; the epoch and the
    flags live on the device, so replays stay correct)."""
    W, H, G, L = 1024, 1024, 4, 4
    ranks = make_ranks(W, H, G, L)
    x = workloads.uniform_real(W, H, 7)
    fill(ranks, x)
    D.sequential_step(ranks)            # warm-up: tensor maps, first launches
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        D.sequential_step(ranks)
    for rep in range(3):
        x = workloads.uniform_real(W, H, 50 + rep)
        fill(ranks, x)
        g.replay()
        torch.cuda.synchronize()
        np.testing.assert_array_equal(gather(ranks, W, H, L), single_gpu(x, L))
    close(ranks)


def test_peer_strip_alone_is_the_single_image_transform():
    """One rank (no neighbour): the concurrent-rank step runs every quad row
    in the INTERIOR launch and publishes nothing."""
    W, H, L = 777, 513, 4
    r = D.PeerStripPyramid(W, H, 0, 1, L, device="cuda")
    r.connect_local([r], dwt2.DWT2_PEER_RANKS)
    x = workloads.uniform_real(W, H, 9)
    fill([r], x)
    r.step()
    torch.cuda.synchronize()
    np.testing.assert_array_equal(gather([r], W, H, L), single_gpu(x, L))
    close([r])


def test_peer_wait_times_out_instead_of_hanging():
    """A BOUNDARY part whose neighbour never published its flag gives up after
    the context's timeout and latches DWT2_ETIMEOUT (no hang)."""
    W, H, G, L = 256, 256, 2, 1
    ranks = make_ranks(W, H, G, L, timeout_ms=50)
    fill(ranks, workloads.uniform_int(W, H, 1))
    r0 = ranks[0]
    r0.ctx.level(0, dwt2.DWT2_STRIP_ALL, r0.out)            # rank 1 never publishes its level 0
    torch.cuda.synchronize()
    assert r0.status() == dwt2.DWT2_ETIMEOUT
    assert ranks[1].status() == dwt2.DWT2_OK
    for r in ranks:
        r.close()


def test_peer_connect_validation():
    W, H, G, L = 128, 128, 2, 2
    ranks = [D.PeerStripPyramid(W, H, g, G, L, device="cuda") for g in range(G)]
    d0, d1 = ranks[0].ctx.export(), ranks[1].ctx.export()
    with pytest.raises(dwt2.DWT2Error):
        ranks[0].ctx.connect(None, None, dwt2.DWT2_PEER_SEQUENTIAL)      # rank 0 has a rank below
    with pytest.raises(dwt2.DWT2Error):
        ranks[0].ctx.connect(d0, d1, dwt2.DWT2_PEER_SEQUENTIAL)          # row 0 has no rank above
    bad = dwt2.PeerDesc.from_bytes(d1.to_bytes())
    bad.levels = 3
    with pytest.raises(dwt2.DWT2Error):
        ranks[0].ctx.connect(None, bad, dwt2.DWT2_PEER_SEQUENTIAL)       # geometry differs
    ranks[0].ctx.connect(None, d1, dwt2.DWT2_PEER_SEQUENTIAL)
    with pytest.raises(dwt2.DWT2Error):
        ranks[0].ctx.forward(ranks[0].out)                                # whole steps: concurrent ranks only
    with pytest.raises(dwt2.DWT2Error):
        ranks[0].ctx.connect(None, d1, dwt2.DWT2_PEER_SEQUENTIAL)        # connect once
    for r in ranks:
        r.close()
