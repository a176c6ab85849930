"""Out-of-bounds checks without compute-sanitizer (closed on this GPU pool):
every kernel family runs on inputs and outputs that sit inside larger
buffers whose surroundings hold NaN (inputs) or a canary pattern (outputs).
A kernel that reads outside its input would pull a NaN into the result (the
oracle comparison then fails); one that writes outside its output would
change a canary.  Inputs must come back unchanged.  Sizes are small and
ragged (odd widths: the bulk-copy loader's clamped first / last bytes; tiny
levels; batch gaps)."""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import dwt2, workloads

pytestmark = pytest.mark.gpu

GUARD = 4099            # floats of guard before and after (not a multiple of 4: misaligned neighbours too)
CANARY = -12345.678


def embed(x: np.ndarray, fill: float, align: int = 0):
    """x inside a flat device buffer [guard | x | guard]; returns (view, buffer).
    align: offset in floats of the image start inside the buffer modulo 4."""
    n = x.size
    pre = GUARD - (GUARD % 4) + align
    buf = torch.full((pre + n + GUARD,), fill, dtype=torch.float32, device="cuda")
    view = buf[pre:pre + n].view(x.shape)
    view.copy_(torch.from_numpy(np.ascontiguousarray(x)))
    return view, buf, pre


def check_guards(buf, pre, n, fill, what):
    b = buf.cpu().numpy()
    before, after = b[:pre], b[pre + n:]
    if np.isnan(fill):
        assert np.isnan(before).all() and np.isnan(after).all(), f"{what}: guard written"
    else:
        assert (before == fill).all() and (after == fill).all(), f"{what}: guard written"


@pytest.mark.parametrize("W,H,L", [(300, 212, 3), (4095, 31, 2), (257, 130, 2), (2, 2, 1), (33, 1000, 5)])
@pytest.mark.parametrize("align", [0, 1, 3])
def test_forward_and_inverse_stay_in_bounds(W, H, L, align):
    x = workloads.uniform_int(W, H, W * H + align)
    xin, bin_, pin = embed(x, np.nan, align)
    out, bout, pout = embed(np.zeros((H, W), np.float32), CANARY, (align + 2) % 4)
    plan = dwt2.Plan(W, H, L)
    plan.forward(xin, out)
    torch.cuda.synchronize()
    check_guards(bout, pout, x.size, CANARY, "forward out")
    check_guards(bin_, pin, x.size, np.nan, "forward in")
    np.testing.assert_array_equal(xin.cpu().numpy(), x)
    ref = oracle.forward(x.astype(np.float64), L, round_f32=True)
    np.testing.assert_array_equal(out.cpu().numpy().astype(np.float64), ref)
    # inverse from the NaN-guarded pyramid into a canary-guarded image
    yin, byin, pyin = embed(out.cpu().numpy(), np.nan, align)
    rec, brec, prec = embed(np.zeros((H, W), np.float32), CANARY, 1)
    plan.inverse(yin, rec)
    torch.cuda.synchronize()
    check_guards(brec, prec, x.size, CANARY, "inverse out")
    if L <= 2:
        np.testing.assert_array_equal(rec.cpu().numpy(), x)
    else:
        assert np.abs(rec.cpu().numpy() - x).max() <= 1e-4
    plan.close()


@pytest.mark.parametrize("wavelet", ["cdf97", "cdf53_k2"])
@pytest.mark.parametrize("scheme", [None, "sep_lifting", "sep_conv", "nonsep_lifting", "nonsep_adapted",
                                    "nonsep_naive"])
def test_k2_and_schemes_stay_in_bounds(wavelet, scheme):
    if scheme is not None and wavelet != "cdf53_k2":
        pytest.skip("schemes run with the 5/3 plan")
    W, H, L = 301, 133, 2
    x = workloads.uniform_int(W, H, 11)
    xin, bin_, pin = embed(x, np.nan, 1)
    out, bout, pout = embed(np.zeros((H, W), np.float32), CANARY, 2)
    if scheme is None:
        plan = dwt2.Plan(W, H, L, wavelet=wavelet)
        plan.forward(xin, out)
        ref = (oracle.forward(x.astype(np.float64), L, wavelet="cdf97") if wavelet == "cdf97"
               else oracle.forward(x.astype(np.float64), L))
    else:
        plan = dwt2.Plan(W, H, L)
        plan.forward_scheme(scheme, xin, out)
        ref = oracle.forward(x.astype(np.float64), L)
    torch.cuda.synchronize()
    check_guards(bout, pout, x.size, CANARY, f"{wavelet} {scheme} out")
    got = out.cpu().numpy().astype(np.float64)
    assert np.isfinite(got).all()
    assert np.abs(got - ref).max() <= 1e-4
    plan.close()


def test_batched_gaps_stay_untouched():
    """Batched calls with image strides larger than the image: the gaps
    between images (NaN in the input, canary in the output) stay as they are."""
    W, H, L, N, gap = 515, 66, 2, 3, 37
    stride = W * H + gap
    xs = [workloads.uniform_int(W, H, 50 + i) for i in range(N)]
    src = torch.full((N * stride,), float("nan"), device="cuda")
    dst = torch.full((N * stride,), CANARY, device="cuda")
    for i, x in enumerate(xs):
        src[i * stride:i * stride + W * H].copy_(torch.from_numpy(x.ravel()))
    plan = dwt2.Plan(W, H, L, max_count=N)
    dwt2.dwt2_forward_batched(plan.handle, src.data_ptr(), dst.data_ptr(), N, stride, stride,
                              torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    d = dst.cpu().numpy()
    for i, x in enumerate(xs):
        np.testing.assert_array_equal(d[i * stride:i * stride + W * H].reshape(H, W).astype(np.float64),
                                      oracle.forward(x.astype(np.float64), L, round_f32=True))
        assert (d[i * stride + W * H:(i + 1) * stride] == CANARY).all()
    plan.close()
