"""Pins for the CPU oracle (-m "not gpu").

The oracle (oracle/dwt53_oracle.c) is checked against what PAPER.md and the
mathematics fix, never against itself:

* hand-derived worked examples (tests/golden/hand_derived.txt);
* the whole-sample symmetric reflection rule on explicit indices;
* closed forms: 2x2 quad, constants (DC gain 1), linear ramps and the
  bilinear xy (two vanishing moments), quadratics x^2, y^2, x^2 y^2;
* the impulse response = tensor products of the analysis taps;
* a library route: numpy reflect-padding + np.convolve (a textbook filter
  bank, Eq. (1)) equals the lifting result;
* lifting (Eq. (2)/(3)) == brute-force convolution (Eq. (1)/(4)) bit for bit
  on every size 1..16 x 1..16 (the schemes compute the
  same transform);
* perfect reconstruction through the independent inverse;
* the exactness bound for integer inputs (coefficients on the 1/64 and
  1/4096 grids) that makes bit-exact GPU parity a requirement.

A plausible oracle bug (dropped term, wrong sign, transposed operand, wrong
phase or boundary) fails at least one of these.
"""
import os

import numpy as np
import pytest

from paper_1708_07853_b200 import workloads

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "hand_derived.txt")


def _golden_cases():
    cases, cur = [], None
    with open(GOLDEN) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, _, rest = line.partition(" ")
            if key == "case":
                cur = {"name": rest}
                cases.append(cur)
            elif key == "kind":
                cur["kind"] = rest
            elif key == "dims":
                cur["W"], cur["H"] = map(int, rest.split())
            elif key in ("in", "out"):
                cur[key] = np.array([float(v) for v in rest.split()])
    return cases


@pytest.mark.parametrize("case", _golden_cases(), ids=lambda c: c["name"])
def test_golden_hand_derived(oracle_mod, case):
    if case["kind"] == "1d":
        got = oracle_mod.fwd_1d(case["in"])
        np.testing.assert_array_equal(got, case["out"])
        np.testing.assert_array_equal(oracle_mod.inv_1d(got), case["in"])
    else:
        img = case["in"].reshape(case["H"], case["W"])
        for alg in ("lifting", "conv"):
            got = oracle_mod.forward(img, 1, algorithm=alg)
            np.testing.assert_array_equal(got.ravel(), case["out"], err_msg=alg)


def test_wss_reflection(oracle_mod):
    # x[-k] = x[k], x[N-1+k] = x[N-1-k]
    expect = {(-1, 5): 1, (-2, 5): 2, (5, 5): 3, (6, 5): 2, (8, 5): 0, (9, 5): 1,
              (-1, 2): 1, (2, 2): 0, (-2, 2): 0, (3, 4): 3, (4, 4): 2, (0, 1): 0, (-3, 1): 0, (7, 1): 0}
    for (k, n), v in expect.items():
        assert oracle_mod.wss_index(k, n) == v, (k, n)


def _grid(W, H):
    y, x = np.mgrid[0:H, 0:W].astype(np.float64)
    return x, y


@pytest.mark.parametrize("W,H", [(1, 1), (1, 7), (2, 2), (3, 5), (16, 12), (17, 13), (33, 8)])
@pytest.mark.parametrize("levels", [1, 2, 3])
def test_constant_image(oracle_mod, W, H, levels):
    c = 117.25
    out = oracle_mod.forward(np.full((H, W), c), levels)
    w, h = W, H
    for _ in range(levels):
        w, h = (w + 1) // 2, (h + 1) // 2
    expect = np.zeros((H, W))
    expect[:h, :w] = c
    np.testing.assert_array_equal(out, expect)


def _bands(out, W, H):
    wl, hl = (W + 1) // 2, (H + 1) // 2
    return out[:hl, :wl], out[:hl, wl:], out[hl:, :wl], out[hl:, wl:]


@pytest.mark.parametrize("W,H", [(16, 12), (17, 13), (20, 9), (9, 20)])
def test_linear_ramps_two_vanishing_moments(oracle_mod, W, H):
    x, y = _grid(W, H)
    alpha, beta, gamma = 1.5, -2.25, 7.0
    for f, name in ((alpha * x + beta * y + gamma, "affine"), (x * y, "bilinear")):
        LL, HL, LH, HH = _bands(oracle_mod.forward(f, 1), W, H)
        ms = np.arange(HL.shape[1])
        ns = np.arange(LH.shape[0])
        inner_m = 2 * ms + 2 <= W - 1          # g1 support inside the image
        inner_n = 2 * ns + 2 <= H - 1
        assert np.all(HL[:, inner_m] == 0), name
        assert np.all(LH[inner_n, :] == 0), name
        assert np.all(HH[:, inner_m] == 0) and np.all(HH[inner_n, :] == 0), name
        # LL interpolates: LL(m, n) = f(2m, 2n) while the 5-tap support stays
        # inside (the WSS mirror of a linear function is symmetric about the
        # edge sample, so m = 0 / n = 0 also qualify).
        mm = np.arange(LL.shape[1])[2 * np.arange(LL.shape[1]) + 2 <= W - 1]
        nn = np.arange(LL.shape[0])[2 * np.arange(LL.shape[0]) + 2 <= H - 1]
        fx = f[2 * nn][:, 2 * mm]
        np.testing.assert_array_equal(LL[np.ix_(nn, mm)], fx, err_msg=name)
    # even sizes: the WSS kink at the right/bottom edge leaves exactly the slope
    f = alpha * x + beta * y + gamma
    LL, HL, LH, HH = _bands(oracle_mod.forward(f, 1), W, H)
    if W % 2 == 0:
        np.testing.assert_array_equal(HL[:, -1], alpha)
    if H % 2 == 0:
        np.testing.assert_array_equal(LH[-1, :], beta)


@pytest.mark.parametrize("W,H", [(16, 16), (19, 15)])
def test_quadratics(oracle_mod, W, H):
    x, y = _grid(W, H)
    # f = x^2: d = (2i+1)^2 - ((2i)^2 + (2i+2)^2)/2 = -1 ; s = 4 i^2 - 1/2
    LL, HL, LH, HH = _bands(oracle_mod.forward(x * x, 1), W, H)
    inner_m = 2 * np.arange(HL.shape[1]) + 2 <= W - 1
    assert np.all(HL[:, inner_m] == -1.0)
    assert np.all(LH == 0) and np.all(HH == 0)
    m = np.arange(LL.shape[1])
    ok = (2 * m - 2 >= 0) & (2 * m + 2 <= W - 1)
    np.testing.assert_array_equal(LL[:, ok], np.broadcast_to(4.0 * m[ok] ** 2 - 0.5, LL[:, ok].shape))
    # f = y^2 -> LH = -1 in the interior
    LL, HL, LH, HH = _bands(oracle_mod.forward(y * y, 1), W, H)
    inner_n = 2 * np.arange(LH.shape[0]) + 2 <= H - 1
    assert np.all(LH[inner_n, :] == -1.0)
    assert np.all(HL == 0) and np.all(HH == 0)
    # f = x^2 y^2 -> HH = (-1)(-1) = +1 in the interior
    LL, HL, LH, HH = _bands(oracle_mod.forward(x * x * y * y, 1), W, H)
    inner_m = 2 * np.arange(HH.shape[1]) + 2 <= W - 1
    inner_n = 2 * np.arange(HH.shape[0]) + 2 <= H - 1
    assert np.all(HH[np.ix_(inner_n, inner_m)] == 1.0)


def test_impulse_response_taps(oracle_mod):
    # Analysis taps of the lifting pair (Eq. (1)-(2)):
    #   h0 = (-1/8, 1/4, 3/4, 1/4, -1/8) around even samples,
    #   g1 = (-1/2, 1, -1/2) around odd samples.
    h0 = {-2: -0.125, -1: 0.25, 0: 0.75, 1: 0.25, 2: -0.125}
    g1 = {-1: -0.5, 0: 1.0, 1: -0.5}
    W, H = 24, 20
    for py, px in [(9, 11), (10, 12), (9, 12), (10, 11)]:
        img = np.zeros((H, W))
        img[py, px] = 1.0
        LL, HL, LH, HH = _bands(oracle_mod.forward(img, 1), W, H)

        def resp(ftx, cx, fty, cy, shape):
            r = np.zeros(shape)
            for n in range(shape[0]):
                for m in range(shape[1]):
                    r[n, m] = ftx.get(px - cx(m), 0.0) * fty.get(py - cy(n), 0.0)
            return r

        ev = lambda k: 2 * k
        od = lambda k: 2 * k + 1
        np.testing.assert_array_equal(LL, resp(h0, ev, h0, ev, LL.shape))
        np.testing.assert_array_equal(HL, resp(g1, od, h0, ev, HL.shape))
        np.testing.assert_array_equal(LH, resp(h0, ev, g1, od, LH.shape))
        np.testing.assert_array_equal(HH, resp(g1, od, g1, od, HH.shape))


def _numpy_filterbank_level(img):
    """Textbook filter bank with library primitives: numpy 'reflect' padding
    is whole-sample symmetric extension; np.convolve filters; keep the even
    phase for the low band and the odd phase for the high band."""
    h0 = np.array([-1, 2, 6, 2, -1], dtype=np.float64) / 8.0
    g1 = np.array([-1, 2, -1], dtype=np.float64) / 2.0

    def rows(a):
        W = a.shape[1]
        p = np.pad(a, ((0, 0), (2, 2)), mode="reflect")
        lo = np.stack([np.convolve(r, h0, mode="valid") for r in p])      # centred on 0..W-1
        hi = np.stack([np.convolve(r, g1, mode="valid")[1:-1] for r in p])  # centred on 0..W-1
        return np.concatenate([lo[:, 0::2], hi[:, 1::2]], axis=1) if W > 1 else a

    t = rows(img)
    return rows(t.T).T


@pytest.mark.parametrize("W,H", [(3, 3), (4, 6), (7, 5), (32, 17), (31, 30)])
def test_library_filterbank(oracle_mod, W, H):
    rng = np.random.default_rng(W * 100 + H)
    img = rng.uniform(-100, 100, size=(H, W))
    ref = _numpy_filterbank_level(img)
    got = oracle_mod.forward(img, 1)
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-12)


def test_lifting_equals_convolution_all_small_sizes(oracle_mod):
    rng = np.random.default_rng(7)
    for H in range(1, 17):
        for W in range(1, 17):
            img = rng.integers(0, 256, size=(H, W)).astype(np.float64)
            a = oracle_mod.forward(img, 1, algorithm="lifting")
            b = oracle_mod.forward(img, 1, algorithm="conv")
            np.testing.assert_array_equal(a, b, err_msg=f"{W}x{H}")


@pytest.mark.parametrize("W,H,levels", [(37, 29, 3), (64, 64, 4), (65, 33, 5), (100, 7, 2)])
def test_lifting_equals_convolution_multilevel(oracle_mod, W, H, levels):
    rng = np.random.default_rng(W + H + levels)
    img = rng.integers(0, 256, size=(H, W)).astype(np.float64)
    for rnd in (False, True):
        a = oracle_mod.forward(img, levels, round_f32=rnd, algorithm="lifting")
        b = oracle_mod.forward(img, levels, round_f32=rnd, algorithm="conv")
        np.testing.assert_array_equal(a, b)


@pytest.mark.parametrize("W,H,levels", [(1, 1, 1), (2, 3, 1), (17, 9, 2), (64, 48, 3), (301, 409, 6),
                                        (1024, 1023, 8)])
def test_perfect_reconstruction(oracle_mod, W, H, levels):
    rng = np.random.default_rng(3)
    img = rng.integers(0, 256, size=(H, W)).astype(np.float64)
    rec = oracle_mod.inverse(oracle_mod.forward(img, levels), levels)
    if levels <= 2:
        np.testing.assert_array_equal(rec, img)
    else:
        np.testing.assert_allclose(rec, img, rtol=0, atol=1e-9)
    real = rng.uniform(0, 255, size=(H, W)).astype(np.float32).astype(np.float64)
    rec = oracle_mod.inverse(oracle_mod.forward(real, levels), levels)
    np.testing.assert_allclose(rec, real, rtol=0, atol=1e-10)


def test_integer_exactness_grid(oracle_mod):
    """Integer pixels in [0, 255]: level-1 coefficients are multiples of 1/64
    with |c| <= 1020, level-2 ones multiples of 1/4096 (< 2^24 ulps), so any
    correct fp32 or fp64 evaluation order is exact -> GPU error must be 0."""
    img = workloads.uniform_int(256, 192, 11).astype(np.float64)
    o1 = oracle_mod.forward(img, 1)
    assert np.all(o1 * 64 == np.round(o1 * 64))
    assert np.abs(o1).max() <= 1020
    o2 = oracle_mod.forward(img, 2)
    assert np.all(o2 * 4096 == np.round(o2 * 4096))
    assert np.abs(o2).max() * 4096 < 2 ** 24
    # so rounding each level to fp32 changes nothing at <= 2 levels
    np.testing.assert_array_equal(oracle_mod.forward(img, 2, round_f32=True), o2)


def test_round_f32_variant_close(oracle_mod):
    img = workloads.smooth_noise(257, 200, 5).astype(np.float64)
    a = oracle_mod.forward(img, 5, round_f32=False)
    b = oracle_mod.forward(img, 5, round_f32=True)
    d = np.abs(a - b).max()
    assert 0 < d < 1e-4


def test_conv_sample_matches_full(oracle_mod):
    img32 = workloads.uniform_real(45, 38, 2)
    full = oracle_mod.forward(img32.astype(np.float64), 1)
    W, H = 45, 38
    wl, hl = (W + 1) // 2, (H + 1) // 2
    bands, ms, ns, exp = [], [], [], []
    for b, (w, h, ox, oy) in enumerate([(wl, hl, 0, 0), (W // 2, hl, wl, 0), (wl, H // 2, 0, hl),
                                         (W // 2, H // 2, wl, hl)]):
        for n in range(h):
            for m in range(w):
                bands.append(b); ms.append(m); ns.append(n); exp.append(full[oy + n, ox + m])
    got32 = oracle_mod.conv_sample(img32, bands, ms, ns)
    got64 = oracle_mod.conv_sample(img32.astype(np.float64), bands, ms, ns)
    np.testing.assert_array_equal(got32, np.array(exp))
    np.testing.assert_array_equal(got64, np.array(exp))
    # strided view (pitch > W)
    big = np.zeros((38, 64), dtype=np.float32)
    big[:, :45] = img32
    np.testing.assert_array_equal(oracle_mod.conv_sample(big[:, :45], bands, ms, ns), np.array(exp))


def test_generators_deterministic_and_ranged():
    a = workloads.uniform_int(64, 32, 1)
    assert a.dtype == np.float32 and a.shape == (32, 64)
    np.testing.assert_array_equal(a, workloads.uniform_int(64, 32, 1))
    assert a.min() >= 0 and a.max() <= 255 and np.all(a == np.round(a))
    s = workloads.smooth_noise(128, 96, 2)
    assert s.dtype == np.float32 and s.min() >= 0 and s.max() <= 255
    np.testing.assert_array_equal(s, workloads.smooth_noise(128, 96, 2))
    assert not np.array_equal(s, workloads.smooth_noise(128, 96, 3))
    assert workloads.level_pixels(8192, 8192, 8) == 89_477_120
    assert workloads.CONFIGS["5"].pixels == 1_466_992_864


# --------------------------------------------------------------------------
# Oracle (ii): where the per-level fp32 rounding happens (DESIGN.md reading
# C-A13: every level's whole output -- LL and the three detail bands -- is
# stored as fp32 before the next level reads its LL).  Pinned against a
# level-by-level composition written here: the pinned one-level oracle (i)
# plus numpy's own fp32 rounding, applied to the region each level owns.
# --------------------------------------------------------------------------
def _f32(a):
    return a.astype(np.float32).astype(np.float64)


def _dims(W, H, L):
    ws, hs = [W], [H]
    for _ in range(L):
        ws.append((ws[-1] + 1) // 2)
        hs.append((hs[-1] + 1) // 2)
    return ws, hs


def _compose_forward(oracle_mod, x, L):
    out = x.copy()
    ws, hs = _dims(x.shape[1], x.shape[0], L)
    for k in range(L):
        region = np.ascontiguousarray(out[:hs[k], :ws[k]])
        out[:hs[k], :ws[k]] = _f32(oracle_mod.forward(region, 1))
    return out


def _compose_inverse(oracle_mod, y, L):
    out = y.copy()
    ws, hs = _dims(y.shape[1], y.shape[0], L)
    for k in range(L - 1, -1, -1):
        region = np.ascontiguousarray(out[:hs[k], :ws[k]])
        out[:hs[k], :ws[k]] = _f32(oracle_mod.inverse(region, 1))
    return out


@pytest.mark.parametrize("W,H", [(60, 50), (37, 29), (64, 64)])
@pytest.mark.parametrize("L", [1, 2, 3])
def test_round_f32_rounds_every_level_output(oracle_mod, W, H, L):
    x = np.random.default_rng(W * 7 + H + L).uniform(0, 255, (H, W)).astype(np.float32).astype(np.float64)
    y = oracle_mod.forward(x, L, round_f32=True)
    # every stored coefficient (every level, every subband) is an fp32 value
    np.testing.assert_array_equal(y, _f32(y))
    # and equals the level-by-level composition with fp32 storage between levels
    np.testing.assert_array_equal(y, _compose_forward(oracle_mod, x, L))
    if L == 1:
        np.testing.assert_array_equal(y, _f32(oracle_mod.forward(x, 1)))
    # the composition is discriminating: rounding only at the end differs
    if L >= 2:
        assert not np.array_equal(y, _f32(oracle_mod.forward(x, L)))


@pytest.mark.parametrize("W,H", [(60, 50), (37, 29)])
@pytest.mark.parametrize("L", [1, 2, 3])
def test_inverse_round_f32_rounds_every_level(oracle_mod, W, H, L):
    rng = np.random.default_rng(W + H * 3 + L)
    # a real-valued fp32 pyramid (not the transform of anything in particular)
    y = rng.uniform(-300, 300, (H, W)).astype(np.float32).astype(np.float64)
    r = oracle_mod.inverse(y, L, round_f32=True)
    np.testing.assert_array_equal(r, _f32(r))
    np.testing.assert_array_equal(r, _compose_inverse(oracle_mod, y, L))
    if L >= 2:
        assert not np.array_equal(r, _f32(oracle_mod.inverse(y, L)))
    # fp64 inverse with per-level rounding still reconstructs a real image to fp32 accuracy
    x = rng.uniform(0, 255, (H, W)).astype(np.float32).astype(np.float64)
    rt = oracle_mod.inverse(oracle_mod.forward(x, L, round_f32=True), L, round_f32=True)
    assert np.abs(rt - x).max() < 1e-4
