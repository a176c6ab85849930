"""The tail kernel (dwt53_tail_kernel: the small last levels of a forward in
one launch, pointwise 5 x 5 analysis filters per quad, a grid barrier between
levels) against the oracle, bit for bit against oracle (ii): sizes at and
around the tail threshold (levels of <= 256^2 input), odd sizes down to 2 x 2,
batches, pyramids that switch from the level kernel to the tail kernel, and
repeated calls / graph replays (the barrier counters reset themselves)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import dwt2, workloads

pytestmark = pytest.mark.gpu


def _levels_max(W, H):
    L = 0
    while W >= 2 and H >= 2:
        W, H, L = (W + 1) // 2, (H + 1) // 2, L + 1
    return L


@pytest.mark.parametrize("W,H", [(2, 2), (3, 2), (2, 3), (3, 3), (5, 7), (33, 17), (255, 257), (256, 256),
                                 (257, 255), (258, 256), (300, 212), (513, 511)])
def test_tail_levels_bit_exact(W, H):
    x = workloads.uniform_real(W, H, W * 3 + H)
    for L in range(1, _levels_max(W, H) + 1):
        plan = dwt2.Plan(W, H, L)
        got = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        plan.close()
        ref = oracle.forward(x.astype(np.float64), L, round_f32=True)
        d = np.abs(got.astype(np.float64) - ref)
        assert not d.any(), f"{W}x{H} L{L}: {int(np.count_nonzero(d))} off, max {d.max()}"


@pytest.mark.parametrize("W,H,L,count", [(64, 64, 3, 5), (255, 129, 4, 3), (100, 300, 6, 2)])
def test_tail_batched(W, H, L, count):
    xs = np.stack([workloads.uniform_real(W, H, 100 + i) for i in range(count)])
    plan = dwt2.Plan(W, H, L, max_count=count)
    got = plan.forward(torch.from_numpy(xs).cuda()).cpu().numpy()
    plan.close()
    for i in range(count):
        ref = oracle.forward(xs[i].astype(np.float64), L, round_f32=True)
        assert np.array_equal(got[i].astype(np.float64), ref), f"image {i}"


def test_tail_repeated_calls_and_graph_replays():
    """Config 4's shape (levels 6-8 on the tail kernel) 30 times in a row and
    as a replayed CUDA graph: every output identical to the first."""
    W = H = 8192
    x = torch.from_numpy(workloads.smooth_noise(W, H, 4)).cuda()
    plan = dwt2.Plan(W, H, 8)
    ref = plan.forward(x).clone()
    out = torch.empty_like(x)
    for _ in range(30):
        plan.forward(x, out)
    torch.cuda.synchronize()
    assert torch.equal(out, ref)
    g = torch.cuda.CUDAGraph()
    outs = [torch.empty_like(x) for _ in range(3)]
    with torch.cuda.graph(g):
        for o in outs:
            plan.forward(x, o)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    for o in outs:
        assert torch.equal(o, ref)
    plan.close()


def test_plan_info_counts_the_tail_launch():
    p = dwt2.Plan(8192, 8192, 8)
    assert p.info().launches_per_forward == 6          # levels 1-5 + one tail launch (levels 6-8)
    p.close()
    p = dwt2.Plan(512, 512, 1)
    assert p.info().launches_per_forward == 1
    p.close()


@pytest.mark.parametrize("W,H", [(2, 2), (3, 5), (64, 64), (255, 257), (1025, 1023)])
def test_tail_k2_cdf97_within_tolerance(W, H):
    """CDF 9/7 plans: the small levels run in the tail kernel with the radius-4
    filters derived from the lifting pair on the host; every level count
    against the fp64 oracle (i) within BASELINE's 1e-4."""
    x = workloads.uniform_real(W, H, W + 7 * H)
    for L in range(1, _levels_max(W, H) + 1):
        plan = dwt2.Plan(W, H, L, wavelet="cdf97")
        got = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        plan.close()
        ref = oracle.forward(x.astype(np.float64), L, round_f32=False, wavelet="cdf97")
        assert np.abs(got - ref).max() <= 1e-4, f"{W}x{H} L{L}"


def test_tail_k2_with_53_pair_bit_identical():
    """The K = 2 path with the CDF 5/3 pair (its tail uses the radius-4 filters
    derived from (-1/2, 1/4, 0, 0), dyadic taps, exact) equals the 5/3 product
    path bit for bit, on a pyramid that ends in the tail."""
    W, H, L = 777, 513, 7
    x = workloads.uniform_real(W, H, 5)
    p53 = dwt2.Plan(W, H, L)
    pk2 = dwt2.Plan(W, H, L, wavelet="cdf53_k2")
    a = p53.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    b = pk2.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    p53.close()
    pk2.close()
    np.testing.assert_array_equal(a, b)
