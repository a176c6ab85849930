"""Pins of the CDF 9/7 oracle (oracle/dwt97_oracle.c)
against things other than itself:

* the published CDF 9/7 analysis filter bank (JPEG 2000 irreversible 9/7):
  algorithm B97 is written from those taps, A97 from the lifting constants,
  so A97 == B97 on every size and level pins the constants, their order,
  signs and the scaling (and the WSS extension, which both apply
  independently);
* the filter bank's own facts: low-pass DC gain 1, high-pass DC gain 0,
  four vanishing moments of the analysis high-pass (f = 1, x, x^2, x^3 give
  zero detail away from the borders);
* perfect reconstruction of the inverse (C97);
* the 1-D impulse response of the lifting equals the printed taps.

Readings (C-B1..C-B3): constants of Daubechies &
Sweldens (1998) with JPEG 2000 normalisation (low / K, high * K).
"""
import numpy as np
import pytest

import oracle

# published analysis taps, written here independently of the C source
H97 = {0: 0.6029490182363579, 1: 0.2668641184428723, 2: -0.07822326652898785, 3: -0.01686411844287495,
       4: 0.02674875741080976}
G97 = {0: 1.115087052456994, 1: -0.5912717631142470, 2: -0.05754352622849957, 3: 0.09127176311424948}


def test_published_taps_dc_gains():
    assert abs(H97[0] + 2 * sum(H97[k] for k in range(1, 5)) - 1.0) < 1e-14
    assert abs(G97[0] + 2 * sum(G97[k] for k in range(1, 4))) < 1e-14


def test_impulse_response_is_published_filter_bank():
    n = 40
    for p in (18, 19):                       # impulse on an even and an odd sample
        x = np.zeros(n)
        x[p] = 1.0
        y = oracle.fwd_1d_97(x)
        low, high = y[:n // 2], y[n // 2:]
        for i in range(n // 2):
            off_l = p - 2 * i                # tap offset seen by low[i] (centred on 2i)
            exp_l = H97.get(abs(off_l), 0.0)
            off_h = p - (2 * i + 1)          # high[i] centred on 2i+1
            exp_h = G97.get(abs(off_h), 0.0)
            assert abs(low[i] - exp_l) < 1e-14, (p, i)
            assert abs(high[i] - exp_h) < 1e-14, (p, i)


def test_lifting_equals_published_convolution_all_small_sizes():
    rng = np.random.default_rng(97)
    for H in range(1, 17):
        for W in range(1, 17):
            x = rng.uniform(0, 255, (H, W))
            a = oracle.forward(x, 1, wavelet="cdf97")
            b = oracle.forward(x, 1, algorithm="conv", wavelet="cdf97")
            assert np.abs(a - b).max() < 1e-10, (W, H)


@pytest.mark.parametrize("W,H,L", [(64, 64, 4), (77, 45, 3), (301, 129, 5), (33, 512, 6)])
def test_lifting_equals_convolution_multilevel(W, H, L):
    x = np.random.default_rng(W * H).uniform(0, 255, (H, W))
    a = oracle.forward(x, L, wavelet="cdf97")
    b = oracle.forward(x, L, algorithm="conv", wavelet="cdf97")
    assert np.abs(a - b).max() < 1e-9


def test_conv_sample_matches_full_conv():
    x = np.random.default_rng(5).uniform(0, 255, (37, 52)).astype(np.float32)
    full = oracle.forward(x.astype(np.float64), 1, algorithm="conv", wavelet="cdf97")
    band = np.array([0, 1, 2, 3, 0, 3, 1, 2])
    m = np.array([0, 25, 0, 25, 13, 0, 7, 25])
    n = np.array([0, 0, 17, 17, 9, 17, 18, 3])
    res = oracle.conv_sample(x, band, m, n, wavelet="cdf97")
    Wq, Hq = 26, 19
    r0 = np.where(band >= 2, Hq, 0) + n
    c0 = np.where(band % 2 == 1, Wq, 0) + m
    np.testing.assert_allclose(res, full[r0, c0], rtol=0, atol=1e-10)


def test_constant_image_dc_gain_one():
    for W, H in [(1, 1), (2, 3), (33, 40), (100, 7)]:
        c = np.full((H, W), 93.25)
        y = oracle.forward(c, 3, wavelet="cdf97")
        w, h = W, H
        for _ in range(3):
            w, h = (w + 1) // 2, (h + 1) // 2
        ll = y[:h, :w]
        assert np.abs(ll - 93.25).max() < 1e-11
        rest = y.copy()
        rest[:h, :w] = 0
        assert np.abs(rest).max() < 1e-11


@pytest.mark.parametrize("deg", [1, 2, 3])
def test_four_vanishing_moments_interior(deg):
    """x^deg (deg <= 3) is annihilated by the 7-tap high-pass away from the
    borders; x^4 is not (the moment count is exactly 4)."""
    W, H = 64, 8
    xs = np.arange(W, dtype=np.float64) / 8.0
    img = np.tile(xs ** deg, (H, 1))
    y = oracle.forward(img, 1, wavelet="cdf97")
    hl = y[:H // 2, W // 2:]
    assert np.abs(hl[:, 3:-3]).max() < 1e-9
    img4 = np.tile(xs ** 4, (H, 1))
    hl4 = oracle.forward(img4, 1, wavelet="cdf97")[:H // 2, W // 2:]
    assert np.abs(hl4[:, 3:-3]).max() > 1e-4


@pytest.mark.parametrize("W,H,L", [(1, 1, 1), (2, 2, 1), (5, 9, 2), (64, 64, 6), (301, 129, 5), (17, 1000, 4)])
def test_perfect_reconstruction(W, H, L):
    x = np.random.default_rng(W + H).uniform(0, 255, (H, W))
    y = oracle.forward(x, L, wavelet="cdf97")
    assert np.abs(oracle.inverse(y, L, wavelet="cdf97") - x).max() < 1e-10
    # 1-D too, every length
    for n in range(1, 30):
        s = np.random.default_rng(n).uniform(-1, 1, n)
        assert np.abs(oracle.inv_1d_97(oracle.fwd_1d_97(s)) - s).max() < 1e-13


def test_round_f32_rounds_every_level():
    x = np.random.default_rng(3).uniform(0, 255, (50, 60))
    y = oracle.forward(x, 2, round_f32=True, wavelet="cdf97")
    assert np.array_equal(y, y.astype(np.float32).astype(np.float64))
    y1 = oracle.forward(x, 1, wavelet="cdf97")
    assert np.array_equal(oracle.forward(x, 1, round_f32=True, wavelet="cdf97"),
                          y1.astype(np.float32).astype(np.float64))


# --------------------------------------------------------------------------
# general K <= 2 lifting oracle (oracle_lift2_forward): pinned by its two
# special cases, each an independently written oracle
# --------------------------------------------------------------------------
C97 = (-1.586134342059924, -0.052980118572961, 0.882911075530934, 0.443506852043971)
K97 = 1.230174104914001


@pytest.mark.parametrize("W,H,L", [(1, 1, 1), (7, 5, 2), (37, 45, 3), (64, 33, 5)])
def test_general_lifting_reduces_to_53_and_97(W, H, L):
    x = np.random.default_rng(W * 31 + H).integers(0, 256, (H, W)).astype(np.float64)
    np.testing.assert_array_equal(oracle.forward_lifting2(x, L, (-0.5, 0.25, 0.0, 0.0), 1.0), oracle.forward(x, L))
    np.testing.assert_array_equal(oracle.forward_lifting2(x, L, C97, K97), oracle.forward(x, L, wavelet="cdf97"))


def test_general_lifting_is_linear_and_scaled():
    """A made-up wavelet: the transform is linear, and K scales low / high as stated."""
    rng = np.random.default_rng(8)
    x, y = rng.uniform(0, 255, (2, 30, 22))
    c = (-0.3, 0.15, 0.1, -0.05)
    f = lambda im, K: oracle.forward_lifting2(im, 1, c, K)
    np.testing.assert_allclose(f(2 * x - 3 * y, 1.0), 2 * f(x, 1.0) - 3 * f(y, 1.0), atol=1e-10)
    a, b = f(x, 1.0), f(x, 2.0)
    # 2-D: LL / K^2, HL and LH * 1, HH * K^2
    np.testing.assert_allclose(b[:15, :11], a[:15, :11] / 4, atol=1e-12)
    np.testing.assert_allclose(b[:15, 11:], a[:15, 11:], atol=1e-12)
    np.testing.assert_allclose(b[15:, 11:], a[15:, 11:] * 4, atol=1e-12)
