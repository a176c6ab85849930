"""CPU checks of bench.py's measurement protocol (no GPU): which workloads
count as L2-sized, how many buffer pairs the timed steps cycle over, and that
the JSON config says so."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1708_07853_b200 import workloads  # noqa: E402

L2 = 126e6


@pytest.mark.parametrize("name", ["1", "2", "3", "4", "4b", "5"])
@pytest.mark.parametrize("steps", [3, 20, 100])
def test_buffer_pairs_keep_every_step_cold(name, steps):
    cfg = workloads.CONFIGS[name]
    pair_bytes = cfg.pixels * 8
    n = bench.buffer_pairs(cfg, steps)
    assert 1 <= n <= max(1, steps)
    if pair_bytes >= 2 * L2:
        assert n == 1                      # inputs larger than the L2: one pair
    elif n < steps:
        # a pair is reused only after more than 2x L2 of other steps' traffic
        assert (n - 1) * pair_bytes > 2 * L2
    else:
        assert n == steps                  # every step its own pair (read once after the flush)
    l2 = bench.describe(cfg, 1, steps)["l2"]
    if pair_bytes < 2 * L2:
        assert f"cycle over {n} input/output pairs" in l2
    else:
        assert "larger than the 126 MB L2" in l2


def test_small_configs_flagged():
    assert bench.buffer_pairs(workloads.CONFIGS["1"], 20) == 20
    assert bench.buffer_pairs(workloads.CONFIGS["2"], 20) == 3
    assert bench.buffer_pairs(workloads.CONFIGS["3"], 20) == 1


# --------------------------------------------------------------------------
# the correctness gate's host logic (bench.gate), on CPU tensors: a stand-in
# runner whose "timed output" is the oracle's own pyramid must pass, and the
# same output with one coefficient moved by one fp32 ulp must fail -- in the
# whole-output mode and in the sampled (border quads + random positions) mode
# --------------------------------------------------------------------------
import types  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402


def _fake_single_runner(cfg, out_np, img):
    r = types.SimpleNamespace()
    r.torch = torch
    r.mode = "single"
    r.nbuf = 2
    r.i = 1
    r.outs = [torch.from_numpy(out_np.copy()), torch.from_numpy(out_np.copy())]
    r.host_img = img
    r.x = torch.from_numpy(img)
    return r


def _args(**kw):
    d = dict(wavelet="cdf53", op="forward", scheme="fused")
    d.update(kw)
    return types.SimpleNamespace(**d)


@pytest.mark.parametrize("full", [True, False])
def test_gate_passes_oracle_output_and_flags_one_ulp(oracle_mod, monkeypatch, full):
    cfg = workloads.Config("t", 1, (workloads.ImageGroup(300, 212, 1, "uniform", 9),), "test")
    img = cfg.groups[0].image(0)
    ref = oracle_mod.forward(img.astype(np.float64), 1, round_f32=True).astype(np.float32)
    if not full:
        monkeypatch.setattr(bench, "GATE_FULL_PX", 0)
    res = bench.gate(_fake_single_runner(cfg, ref, img), cfg, _args())
    assert res["status"] == "pass", res
    assert res["elements_checked"] >= (300 * 212 if full else 4 * bench.GATE_RANDOM)
    # a border coefficient (HH at quad (0, last row)) one ulp off
    bad = ref.copy()
    r, c = 211 // 2 + 105, 150 + 0
    bad[r, c] = np.nextafter(bad[r, c], np.float32(np.inf))
    res = bench.gate(_fake_single_runner(cfg, bad, img), cfg, _args())
    assert res["status"] == "fail" and "bit-exact" in res["error"], res


def test_gate_positions_cover_every_border_and_strip_edges():
    rng = np.random.default_rng(0)
    W, H = 101, 64
    b, m, n = bench._positions(W, H, [0, 1, 2, 3], rng)
    for band, (_, _, rows, cols) in enumerate(bench._bands1(W, H)):
        sel = b == band
        for col in (0, 1, cols - 2, cols - 1):
            assert set(range(rows)) <= set(n[sel & (m == col)])
        for row in (0, 1, rows - 2, rows - 1):
            assert set(range(cols)) <= set(m[sel & (n == row)])
    # a strip's quad rows [10, 20): only those rows, including its own first / last two
    b, m, n = bench._positions(W, H, [1, 3], rng, 10, 20)
    assert n.min() >= 10 and n.max() < 20
    for row in (10, 11, 18, 19):
        assert set(range(W // 2)) <= set(m[(b == 3) & (n == row)])


@pytest.mark.parametrize("wavelet,L", [("cdf53", 3), ("cdf97", 2)])
def test_gate_inverse_against_oracle(oracle_mod, wavelet, L):
    """Inverse gate: the timed output is compared with the oracle's inverse of
    the timed pyramid (bit-exact for 5/3, 1e-4 for 9/7); the round trip is a
    separate, looser sanity bound."""
    cfg = workloads.Config("t", L, (workloads.ImageGroup(130, 97, 1, "smooth", 3),), "test")
    img = cfg.groups[0].image(0)
    pyr = oracle_mod.forward(img.astype(np.float64), L, round_f32=True, wavelet=wavelet).astype(np.float32)
    rec = oracle_mod.inverse(pyr.astype(np.float64), L, round_f32=(wavelet == "cdf53"),
                             wavelet=wavelet).astype(np.float32)
    r = _fake_single_runner(cfg, rec, img)
    r.x = torch.from_numpy(pyr)
    res = bench.gate(r, cfg, _args(wavelet=wavelet, op="inverse"))
    assert res["status"] == "pass", res
    bad = rec.copy()
    bad[50, 60] += 1e-3
    r = _fake_single_runner(cfg, bad, img)
    r.x = torch.from_numpy(pyr)
    assert bench.gate(r, cfg, _args(wavelet=wavelet, op="inverse"))["status"] == "fail"


@pytest.mark.parametrize("L,G", [(1, 2), (1, 3), (3, 4)])
def test_gate_strip_rank_outputs(oracle_mod, L, G):
    """Row-strip mode (bench --gpus N): every rank's strip-local Mallat output,
    cut from the oracle's global pyramid, passes the per-rank gate (level-1
    coefficients of its own quad rows, incl. its first / last two), and one
    ulp moved in a strip's edge quad row fails it."""
    from paper_1708_07853_b200 import distributed as D
    W, H = 200, 96
    cfg = workloads.Config("t", L, (workloads.ImageGroup(W, H, 1, "uniform", 4),), "test")
    img = cfg.groups[0].image(0)
    full = oracle_mod.forward(img.astype(np.float64), L, round_f32=True).astype(np.float32)
    lvl1 = oracle_mod.forward(img.astype(np.float64), 1, round_f32=True).astype(np.float32)
    Wq, Hq, Hh = (W + 1) // 2, (H + 1) // 2, H // 2
    for g in range(G):
        r0, r1 = D.strip_rows_levels(H, g, G, L)
        qs, qe = r0 // 2, (r1 + 1) // 2
        hq_loc = qe - qs
        out = np.zeros((r1 - r0, W), np.float32)
        out[:hq_loc, Wq:] = full[qs:qe, Wq:]                        # HL
        if L == 1:
            out[:hq_loc, :Wq] = full[qs:qe, :Wq]                    # LL
        h0, h1 = min(qs, Hh), min(qe, Hh)
        out[hq_loc:hq_loc + (h1 - h0), :] = full[Hq + h0:Hq + h1, :]   # LH | HH
        np.testing.assert_array_equal(out[:hq_loc, Wq:], lvl1[qs:qe, Wq:])
        r = types.SimpleNamespace(torch=torch, mode="strip", out=torch.from_numpy(out), host_img=img,
                                  ex=types.SimpleNamespace(r0=r0, r1=r1))
        res = bench.gate(r, cfg, _args())
        assert res["status"] == "pass", (g, res)
        bad = out.copy()
        bad[hq_loc - 1, Wq + 3] = np.nextafter(bad[hq_loc - 1, Wq + 3], np.float32(np.inf))   # HL, last own row
        r.out = torch.from_numpy(bad)
        assert bench.gate(r, cfg, _args())["status"] == "fail", g
