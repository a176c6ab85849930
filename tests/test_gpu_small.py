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
