"""The small-level kernel (csrc/tail.cu dwt53_small_kernel): whole levels of
at most 2^16 quads over all images, outside the tail launch (config 1:
512^2), one CTA per 32 x 8 quad block staged in shared memory in one round
of loads, each thread one quad with the exact 5 x 5 analysis filters.  Must be
bit-exact against oracle (ii) (and exact against oracle (i) for integer
inputs at one level) on block-ragged shapes, batches and graph replays."""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import dwt2, workloads

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("W,H", [(2, 2), (3, 3), (5, 2), (63, 17), (64, 16), (65, 15), (130, 97), (300, 212),
                                 (511, 513), (512, 512), (1023, 127), (257, 500)])
@pytest.mark.parametrize("L", [1, 2, 4])
def test_small_levels_bit_exact(W, H, L):
    w, h = W, H
    for _ in range(L - 1):
        w, h = (w + 1) // 2, (h + 1) // 2
    if min(w, h) < 2:
        pytest.skip("a level below 2 x 2")
    x = workloads.uniform_real(W, H, 7 * W + H + L)
    plan = dwt2.Plan(W, H, L)
    got = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    plan.close()
    ref = oracle.forward(x.astype(np.float64), L, round_f32=True)
    np.testing.assert_array_equal(got, ref.astype(np.float32))


def test_config1_integer_exact_against_fp64_oracle():
    x = workloads.uniform_int(512, 512, 1)
    plan = dwt2.Plan(512, 512, 1)
    got = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy().astype(np.float64)
    plan.close()
    assert np.array_equal(got, oracle.forward(x.astype(np.float64), 1))


@pytest.mark.parametrize("W,H,n", [(100, 60, 10), (256, 256, 1), (33, 257, 7)])
def test_small_levels_batched(W, H, n):
    xs = np.stack([workloads.uniform_real(W, H, 3 + i) for i in range(n)])
    plan = dwt2.Plan(W, H, 3, max_count=n)
    got = plan.forward(torch.from_numpy(xs).cuda()).cpu().numpy()
    plan.close()
    for i in range(n):
        ref = oracle.forward(xs[i].astype(np.float64), 3, round_f32=True)
        np.testing.assert_array_equal(got[i], ref.astype(np.float32))


def test_small_level_graph_replays_with_new_inputs():
    W, H = 512, 512
    plan = dwt2.Plan(W, H, 1)
    x = torch.zeros((H, W), device="cuda")
    y = torch.empty_like(x)
    plan.forward(x, y)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        plan.forward(x, y)
    for s in range(3):
        xs = workloads.uniform_real(W, H, 40 + s)
        x.copy_(torch.from_numpy(xs))
        g.replay()
        torch.cuda.synchronize()
        ref = oracle.forward(xs.astype(np.float64), 1, round_f32=True)
        np.testing.assert_array_equal(y.cpu().numpy(), ref.astype(np.float32))
    plan.close()


# ---- the small-level inverse kernel (csrc/tail.cu dwt_small_inv_kernel): small
# levels of an inverse (CDF 5/3: <= 2^16 quads, <= 2^20 when the Mallat pitch is
# not 16-byte aligned; K = 2 wavelets: <= 2^16) by staged pointwise synthesis

@pytest.mark.parametrize("W,H,L", [(2, 2, 1), (3, 5, 1), (64, 16, 2), (65, 17, 3), (130, 97, 4), (300, 212, 3),
                                   (511, 513, 2), (512, 512, 1), (1023, 127, 3), (1025, 1023, 5)])
def test_small_inverse_53_bit_exact(W, H, L):
    """5/3: the pyramid of oracle (ii) is reconstructed bit for bit like oracle (ii)'s inverse."""
    x = workloads.uniform_real(W, H, 5 * W + H + L)
    pyr = oracle.forward(x.astype(np.float64), L, round_f32=True).astype(np.float32)
    plan = dwt2.Plan(W, H, L)
    got = plan.inverse(torch.from_numpy(pyr).cuda()).cpu().numpy()
    plan.close()
    ref = oracle.inverse(pyr.astype(np.float64), L, round_f32=True)
    np.testing.assert_array_equal(got, ref.astype(np.float32))


@pytest.mark.parametrize("W,H,L", [(64, 64, 3), (255, 257, 4), (600, 401, 5), (1024, 1024, 6)])
def test_small_inverse_97_within_tolerance(W, H, L):
    x = workloads.smooth_noise(W, H, W + L)
    plan = dwt2.Plan(W, H, L, wavelet="cdf97")
    pyr = plan.forward(torch.from_numpy(x).cuda())
    got = plan.inverse(pyr).cpu().numpy().astype(np.float64)
    ref = oracle.inverse(pyr.cpu().numpy().astype(np.float64), L, wavelet="cdf97")
    plan.close()
    assert float(np.abs(got - ref).max()) <= 1e-4
    assert float(np.abs(got - x).max()) <= 1e-3        # the round trip


def test_small_inverse_batched_53():
    W, H, L, n = 200, 150, 3, 6
    xs = np.stack([workloads.uniform_real(W, H, 60 + i) for i in range(n)])
    pyrs = np.stack([oracle.forward(xs[i].astype(np.float64), L, round_f32=True) for i in range(n)]).astype(np.float32)
    plan = dwt2.Plan(W, H, L, max_count=n)
    got = plan.inverse(torch.from_numpy(pyrs).cuda()).cpu().numpy()
    plan.close()
    for i in range(n):
        ref = oracle.inverse(pyrs[i].astype(np.float64), L, round_f32=True)
        np.testing.assert_array_equal(got[i], ref.astype(np.float32))
