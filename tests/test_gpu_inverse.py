"""GPU inverse against the CPU oracle's inverse
(algorithm C, oracle/dwt53_oracle.c) and as a round trip through the GPU
forward.

Tolerances (C-A13): the inverse of one level from fp32
coefficients is exact in fp64 (dyadic steps, < 53 bits), so every stored
pixel is the correctly rounded fp32 of the oracle's value -> bit-exact
against oracle(ii) (fp64, each level's reconstruction rounded to fp32), and
within 1e-4 of the fp64-throughout oracle(i).  Integer-valued images at <= 2
levels survive forward + inverse bit for bit.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import dwt2, workloads
from tests._parity import compare

pytestmark = pytest.mark.gpu


def gpu_inverse(y: np.ndarray, levels: int) -> np.ndarray:
    H, W = y.shape
    plan = dwt2.Plan(W, H, levels)
    out = plan.inverse(torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32)).cuda())
    res = out.cpu().numpy()
    plan.close()
    return res


def coeffs_of(x: np.ndarray, levels: int) -> np.ndarray:
    """A realistic fp32 pyramid: the oracle forward, stored as fp32."""
    return oracle.forward(x.astype(np.float64), levels, round_f32=True).astype(np.float32)


def check_inverse(y: np.ndarray, levels: int, what: str):
    got = gpu_inverse(y, levels)
    y64 = y.astype(np.float64)
    ref_ii = oracle.inverse(y64, levels, round_f32=True)
    ref_i = oracle.inverse(y64, levels, round_f32=False)
    st = compare(got, ref_i, ref_ii, False, what)
    if levels == 1:
        d = np.abs(got.astype(np.float64) - ref_ii)
        assert not d.any(), f"{what}: {int(np.count_nonzero(d))} pixels not bit-exact vs oracle(ii), max {d.max()}"
    return st


def test_inverse_tiny_sizes_bit_exact():
    rng = np.random.default_rng(11)
    for H in range(2, 34):
        for W in range(2, 34):
            x = rng.integers(0, 256, size=(H, W)).astype(np.float32)
            y = coeffs_of(x, 1)
            check_inverse(y, 1, f"inv {W}x{H} L1")
            # random (non-transform) coefficients exercise every operand
            r = rng.uniform(-300, 300, size=(H, W)).astype(np.float32)
            check_inverse(r, 1, f"inv random {W}x{H} L1")


@pytest.mark.parametrize("W,H,levels", [
    (1000, 777, 1), (1024, 1024, 2), (1030, 515, 3), (2050, 130, 2), (4095, 301, 3),
    (513, 1025, 4), (2048, 37, 1), (64, 4000, 5), (3001, 4095, 3), (1536, 1537, 6), (130, 2050, 2)])
@pytest.mark.parametrize("kind", ["uniform", "smooth"])
def test_inverse_ragged(W, H, levels, kind):
    x = workloads.GENERATORS[kind](W, H, W * 5 + H)
    y = coeffs_of(x, levels)
    check_inverse(y, levels, f"inv {kind} {W}x{H} L{levels}")


@pytest.mark.parametrize("W,H,levels", [(512, 512, 1), (1027, 514, 2), (4096, 4096, 2), (333, 4097, 2)])
def test_round_trip_integer_exact(W, H, levels):
    """GPU forward then GPU inverse returns integer images bit for bit."""
    x = workloads.uniform_int(W, H, 77 + W)
    plan = dwt2.Plan(W, H, levels)
    xt = torch.from_numpy(x).cuda()
    rec = plan.inverse(plan.forward(xt)).cpu().numpy()
    plan.close()
    np.testing.assert_array_equal(rec, x)


def test_round_trip_config4_tolerance():
    """8 levels of smooth+noise 8193^2 (odd every level): forward + inverse on
    the GPU reconstructs within 1e-4 (fp32 storage of every level)."""
    W = H = 8193
    x = workloads.smooth_noise(W, H, 4)
    plan = dwt2.Plan(W, H, 8)
    xt = torch.from_numpy(x).cuda()
    rec = plan.inverse(plan.forward(xt))
    err = float((rec - xt).abs().max())
    plan.close()
    assert err <= 1e-4, err


def test_inverse_batched_matches_single():
    W, H, L, N = 515, 263, 3, 5
    xs = np.stack([workloads.uniform_real(W, H, 900 + i) for i in range(N)])
    ys = np.stack([coeffs_of(x, L) for x in xs])
    plan = dwt2.Plan(W, H, L, max_count=N)
    got = plan.inverse(torch.from_numpy(ys).cuda()).cpu().numpy()
    plan.close()
    for i in range(N):
        np.testing.assert_array_equal(got[i], gpu_inverse(ys[i], L))


def test_inverse_full_size_config3_sampled():
    """16384^2 (config 3 size): inverse of the integer image's pyramid is the image."""
    W = H = 16384
    x = workloads.uniform_int(W, H, 3)
    plan = dwt2.Plan(W, H, 1)
    xt = torch.from_numpy(x).cuda()
    y = plan.forward(xt)
    rec = plan.inverse(y)
    assert torch.equal(rec, xt)
    plan.close()


def test_inverse_rejects_strip_and_overlap():
    plan = dwt2.Plan(64, 64, 1)
    t = torch.zeros(64, 64, device="cuda")
    with pytest.raises(dwt2.DWT2Error):
        dwt2.dwt2_inverse(plan.handle, t.data_ptr(), t.data_ptr(), 0)
    plan.close()
    sp = dwt2.StripPlan(64, 128, 0, 64)
    buf = torch.zeros(65, 64, device="cuda")
    out = torch.zeros(64, 64, device="cuda")
    with pytest.raises(dwt2.DWT2Error):
        dwt2.dwt2_inverse(sp._p, buf.data_ptr(), out.data_ptr(), 0)
    sp.close()


@pytest.mark.parametrize("W,H,L,N", [(512, 264, 3, 3), (1024, 40, 2, 2), (256, 1000, 4, 4)])
def test_inverse_batched_ring_path(W, H, L, N):
    """Widths with 16-byte aligned subband planes take the cp.async ring
    kernel (levels whose planes stay aligned); batched pyramids against the
    oracle, image by image."""
    xs = np.stack([workloads.uniform_real(W, H, 70 + i) for i in range(N)])
    ys = np.stack([coeffs_of(x, L) for x in xs])
    plan = dwt2.Plan(W, H, L, max_count=N)
    got = plan.inverse(torch.from_numpy(ys).cuda()).cpu().numpy()
    plan.close()
    for i in range(N):
        y64 = ys[i].astype(np.float64)
        compare(got[i], oracle.inverse(y64, L), oracle.inverse(y64, L, round_f32=True), False, f"ring batch {i}")
