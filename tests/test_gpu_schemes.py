"""GPU parity of the paper's comparison schemes (
the fused kernel with Eq. 5's literal operators and with Fig. 3's adapted
arithmetic too;
csrc/schemes.cu): separable lifting (Eq. 3, 4 kernels), separable
convolution (Eq. 4, 2 kernels), non-separable lifting (Eq. 5, 2 kernels),
the adapted scheme (Fig. 3, 2 kernels) and Eq. 5 as one plain kernel -- all
against the CPU oracle on the same seeded inputs.

Tolerances (C-A13): the schemes store fp32 between
steps, so on integer-valued inputs at <= 2 levels every intermediate is on
the 1/64 (1/4096) grid and the result is bit-exact; otherwise the bar is
BASELINE.json's 1e-4 against the fp64 oracle(i).
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import dwt2, workloads
from tests._parity import TOL_I

pytestmark = pytest.mark.gpu

STEP_SCHEMES = ["nonsep_naive", "nonsep_lifting", "nonsep_adapted", "sep_conv", "sep_lifting", "fused_literal",
                "fused_adapted"]


def run_scheme(scheme, x: np.ndarray, levels: int) -> np.ndarray:
    H, W = x.shape[-2:]
    n = 1 if x.ndim == 2 else x.shape[0]
    plan = dwt2.Plan(W, H, levels, max_count=n)
    out = plan.forward_scheme(scheme, torch.from_numpy(np.ascontiguousarray(x)).cuda()).cpu().numpy()
    plan.close()
    return out


def check(scheme, x, levels, exact, what):
    got = run_scheme(scheme, x, levels).astype(np.float64)
    ref = oracle.forward(x.astype(np.float64), levels, round_f32=False)
    err = float(np.abs(got - ref).max())
    if exact:
        assert err == 0.0, f"{scheme} {what}: max abs {err} (expected bit-exact)"
    assert err <= TOL_I, f"{scheme} {what}: max abs {err} > {TOL_I}"
    return err


def test_steps_per_scheme():
    assert [dwt2.dwt2_scheme_steps(dwt2.SCHEMES[s]) for s in ["fused"] + STEP_SCHEMES] == [1, 1, 2, 2, 2, 4, 1, 1]
    with pytest.raises(dwt2.DWT2Error):
        dwt2.dwt2_scheme_steps(99)


@pytest.mark.parametrize("scheme", STEP_SCHEMES)
def test_scheme_tiny_sizes_bit_exact(scheme):
    rng = np.random.default_rng(5)
    for H in range(2, 20):
        for W in range(2, 20):
            x = rng.integers(0, 256, size=(H, W)).astype(np.float32)
            check(scheme, x, 1, True, f"{W}x{H} L1")
    for W, H, L in [(5, 7, 2), (16, 16, 3), (17, 31, 4), (33, 32, 2)]:
        x = rng.integers(0, 256, size=(H, W)).astype(np.float32)
        check(scheme, x, L, L <= 2, f"{W}x{H} L{L}")


@pytest.mark.parametrize("scheme", STEP_SCHEMES)
@pytest.mark.parametrize("W,H,levels,kind", [
    (1000, 777, 1, "uniform"), (1030, 515, 2, "uniform"), (4095, 301, 3, "smooth"),
    (513, 1025, 4, "uniform_real"), (2048, 2048, 2, "uniform"), (1537, 1536, 6, "smooth")])
def test_scheme_ragged(scheme, W, H, levels, kind):
    x = workloads.GENERATORS[kind](W, H, W + 3 * H)
    check(scheme, x, levels, kind == "uniform" and levels <= 2, f"{kind} {W}x{H} L{levels}")


@pytest.mark.parametrize("scheme", STEP_SCHEMES)
def test_scheme_equals_fused_on_config3_size(scheme):
    """16384^2 integer image (config 3): every scheme reproduces the fused
    product path bit for bit (both are exact at one level)."""
    W = H = 16384
    x = torch.from_numpy(workloads.uniform_int(W, H, 3)).cuda()
    plan = dwt2.Plan(W, H, 1)
    ref = plan.forward(x)
    got = plan.forward_scheme(scheme, x)
    assert torch.equal(ref, got)
    plan.close()


@pytest.mark.parametrize("scheme", STEP_SCHEMES)
def test_scheme_batched(scheme):
    W, H, L, N = 301, 130, 3, 4
    xs = np.stack([workloads.uniform_int(W, H, 40 + i) for i in range(N)])
    got = run_scheme(scheme, xs, L)
    for i in range(N):
        np.testing.assert_array_equal(got[i], run_scheme(scheme, xs[i], L))
