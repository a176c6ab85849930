"""Row pitches that are not a multiple of 16 bytes (csrc/dwt2.cu, row-grouped
TMA loader): G = 2 rows (pitch = 8 mod 16 bytes) or
G = 4 rows (odd pitch) form one tensor-map row; the < G rows past the last
whole group are copied by the warp.  Every case is checked against the CPU
oracle, and the other loaders for the same data (batched images with a gap
between them and unaligned base pointers take the bulk-copy loader) must
agree bit for bit."""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import dwt2, workloads
from tests._parity import compare

pytestmark = pytest.mark.gpu


def oracle_pair(x, L):
    x64 = x.astype(np.float64)
    return oracle.forward(x64, L, round_f32=False), oracle.forward(x64, L, round_f32=True)


@pytest.mark.parametrize("W", [4093, 4094, 4095, 4097, 4098, 4099])
def test_widths_mod4_every_tail(W):
    """Heights 2..9, 17, 31, 64: every count of rows past the last whole group
    (H mod G), one level, integer input -> bit-exact against the fp64 oracle."""
    for H in list(range(2, 10)) + [17, 31, 64]:
        x = workloads.uniform_int(W, H, W + H)
        plan = dwt2.Plan(W, H, 1)
        got = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
        plan.close()
        ref_i, ref_ii = oracle_pair(x, 1)
        compare(got, ref_i, ref_ii, True, f"{W}x{H}")


@pytest.mark.parametrize("W,H,L", [(8193, 257, 4), (4094, 1027, 3), (1027, 1025, 6), (6, 4099, 2)])
def test_multilevel_odd_pitch(W, H, L):
    x = workloads.uniform_real(W, H, 3 * W + H)
    plan = dwt2.Plan(W, H, L)
    got = plan.forward(torch.from_numpy(x).cuda()).cpu().numpy()
    plan.close()
    ref_i, ref_ii = oracle_pair(x, L)
    st = compare(got, ref_i, ref_ii, False, f"{W}x{H} L{L}")
    assert st["mismatch_ii"] == 0


@pytest.mark.parametrize("W,H,n", [(37, 29, 5), (4095, 33, 3), (6, 5, 7), (4094, 3, 9)])
def test_batched_contiguous_and_gapped(W, H, n):
    """Contiguous images (one row-grouped tensor map over all n * H rows; the
    group boundaries cross image boundaries) against the oracle, and against
    the same images stored with a gap of 3 floats between them (bulk-copy
    loader)."""
    xs = np.stack([workloads.uniform_int(W, H, 100 + i) for i in range(n)])
    plan = dwt2.Plan(W, H, 2, max_count=n)
    got = plan.forward(torch.from_numpy(xs).cuda()).cpu().numpy()
    for i in range(n):
        ref_i, ref_ii = oracle_pair(xs[i], 2)
        compare(got[i], ref_i, ref_ii, True, f"{W}x{H} image {i} of {n}")
    img = W * H
    stride = img + 3
    gin = torch.full((n * stride,), float("nan"), device="cuda")
    for i in range(n):
        gin[i * stride:i * stride + img] = torch.from_numpy(xs[i].ravel()).cuda()
    gout = torch.empty((n * stride,), device="cuda")
    dwt2.dwt2_forward_batched(plan._p, gin.data_ptr(), gout.data_ptr(), n, stride, stride, 0)
    torch.cuda.synchronize()
    g = gout.cpu().numpy()
    for i in range(n):
        np.testing.assert_array_equal(g[i * stride:i * stride + img].reshape(H, W), got[i])
    plan.close()


@pytest.mark.parametrize("W,H", [(4095, 301), (8194, 64)])
def test_unaligned_base_matches(W, H):
    """The same image at a 4-byte-misaligned address (bulk-copy loader) gives
    the row-grouped result bit for bit."""
    x = workloads.uniform_real(W, H, 9)
    plan = dwt2.Plan(W, H, 3)
    ref = plan.forward(torch.from_numpy(x).cuda())
    buf = torch.empty(W * H + 1, device="cuda")
    xin = buf[1:].view(H, W)
    xin.copy_(torch.from_numpy(x))
    got = plan.forward(xin)
    assert torch.equal(got, ref)
    plan.close()


# --------------------------------------------------------------------------
# inverse: the unaligned ring (csrc/inverse.cu, UA: 19 chunks per plane row
# from the 16-byte boundary below the window, per-plane row shifts)
# --------------------------------------------------------------------------

def _inverse(y, L, n=1):
    H, W = y.shape[-2:]
    plan = dwt2.Plan(W, H, L, max_count=n)
    got = plan.inverse(torch.from_numpy(np.ascontiguousarray(y, dtype=np.float32)).cuda()).cpu().numpy()
    plan.close()
    return got


@pytest.mark.parametrize("W", [4093, 4094, 4095, 4097, 4098, 4099])
def test_inverse_widths_mod4(W):
    """Random coefficients (every operand exercised), one level: bit-exact
    against oracle(ii) for every height class."""
    rng = np.random.default_rng(W)
    for H in list(range(2, 10)) + [17, 64]:
        y = rng.uniform(-300, 300, size=(H, W)).astype(np.float32)
        got = _inverse(y, 1)
        ref = oracle.inverse(y.astype(np.float64), 1, round_f32=True)
        d = np.abs(got.astype(np.float64) - ref)
        assert not d.any(), f"inverse {W}x{H}: {int(np.count_nonzero(d))} pixels off, max {d.max()}"


@pytest.mark.parametrize("W,H,L", [(8193, 257, 4), (4094, 1027, 3), (1027, 1025, 6)])
def test_inverse_multilevel_odd_round_trip(W, H, L):
    """forward then inverse on the GPU, odd pitches at every level: the
    original image within fp32 rounding of a round trip, and against oracle(ii)."""
    x = workloads.uniform_real(W, H, W + 7 * H)
    plan = dwt2.Plan(W, H, L)
    xt = torch.from_numpy(x).cuda()
    y = plan.forward(xt)
    rec = plan.inverse(y).cpu().numpy()
    plan.close()
    assert np.abs(rec.astype(np.float64) - x).max() < 1e-3
    ref = oracle.inverse(y.cpu().numpy().astype(np.float64), L, round_f32=True)
    st = compare(rec, oracle.inverse(y.cpu().numpy().astype(np.float64), L, round_f32=False), ref, False,
                 f"inverse {W}x{H} L{L}")
    assert st["mismatch_ii"] == 0


@pytest.mark.parametrize("W,H,n", [(37, 29, 5), (4095, 33, 3)])
def test_inverse_batched_odd_and_misaligned(W, H, n):
    """Batched odd-size pyramids (UA ring) equal the single-image results,
    and a 4-byte-misaligned pyramid (LDG kernel) gives the same pixels."""
    rng = np.random.default_rng(W + n)
    ys = rng.uniform(-300, 300, size=(n, H, W)).astype(np.float32)
    got = _inverse(ys, 2, n)
    for i in range(n):
        np.testing.assert_array_equal(got[i], _inverse(ys[i], 2))
    plan = dwt2.Plan(W, H, 2)
    buf = torch.empty(W * H + 1, device="cuda")
    yin = buf[1:].view(H, W)
    yin.copy_(torch.from_numpy(ys[0]))
    np.testing.assert_array_equal(plan.inverse(yin).cpu().numpy(), got[0])
    plan.close()
