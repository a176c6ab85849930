"""GPU parity: the CUDA path (through the C ABI binding) against the CPU oracle.

All inputs are seeded synthetic images (paper_1708_07853_b200.workloads).
Sizes span several CTA tiles (512-px groups, 16-row stages) with ragged tails,
odd widths/heights (generic loader path and odd-size WSS rules) and the five
BASELINE.json configs at full size in the launch configuration bench.py uses.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_1708_07853_b200 import dwt2, workloads
from tests._parity import compare, gather, sample_positions, ulp32

pytestmark = pytest.mark.gpu


def gpu_forward(x: np.ndarray, levels: int) -> np.ndarray:
    H, W = x.shape
    plan = dwt2.Plan(W, H, levels)
    out = plan.forward(torch.from_numpy(x).cuda())
    res = out.cpu().numpy()
    plan.close()
    return res


def check(x: np.ndarray, levels: int, exact: bool, what: str):
    got = gpu_forward(x, levels)
    x64 = x.astype(np.float64)
    ref_ii = oracle.forward(x64, levels, round_f32=True)
    ref_i = oracle.forward(x64, levels, round_f32=False)
    return compare(got, ref_i, ref_ii, exact, what)


# --------------------------------------------------------------------------
# small and ragged sizes
# --------------------------------------------------------------------------

def test_all_tiny_sizes_bit_exact():
    """Every W, H in 2..33 (odd/even, widths below one slab, generic and TMA
    loaders), 1 level, plus the deepest valid pyramid on a subset."""
    rng = np.random.default_rng(1)
    for H in range(2, 34):
        for W in range(2, 34):
            x = rng.integers(0, 256, size=(H, W)).astype(np.float32)
            check(x, 1, True, f"{W}x{H} L1")
    for W, H in [(4, 4), (5, 7), (8, 9), (16, 16), (17, 31), (32, 33), (33, 32)]:
        L = 1
        w, h = W, H
        while (w + 1) // 2 >= 2 and (h + 1) // 2 >= 2 and L < 5:
            w, h, L = (w + 1) // 2, (h + 1) // 2, L + 1
        x = rng.integers(0, 256, size=(H, W)).astype(np.float32)
        check(x, L, L <= 2, f"{W}x{H} L{L}")


@pytest.mark.parametrize("W,H,levels", [
    (1000, 777, 1), (1024, 1024, 2), (1030, 515, 3), (2050, 130, 2), (4095, 301, 3),
    (513, 1025, 4), (2048, 37, 1), (64, 4000, 5), (3001, 4095, 3), (1536, 1537, 6)])
@pytest.mark.parametrize("kind", ["uniform", "uniform_real", "smooth"])
def test_ragged_sizes(W, H, levels, kind):
    x = workloads.GENERATORS[kind](W, H, W * 7 + H)
    exact = kind == "uniform" and levels <= 2
    st = check(x, levels, exact, f"{kind} {W}x{H} L{levels}")
    assert st["mismatch_ii"] == 0 or not exact


def test_constant_and_ramp_properties():
    W, H = 1027, 514
    c = np.full((H, W), 93.5, dtype=np.float32)
    out = gpu_forward(c, 3)
    w, h = W, H
    for _ in range(3):
        w, h = (w + 1) // 2, (h + 1) // 2
    exp = np.zeros((H, W), np.float32)
    exp[:h, :w] = 93.5
    np.testing.assert_array_equal(out, exp)
    y, xg = np.mgrid[0:H, 0:W].astype(np.float32)
    f = (0.5 * xg - 0.25 * y + 3.0).astype(np.float32)
    out = gpu_forward(f, 1)
    hl = out[:(H + 1) // 2, (W + 1) // 2:]
    inner = 2 * np.arange(hl.shape[1]) + 2 <= W - 1
    assert np.all(hl[:, inner] == 0)


# --------------------------------------------------------------------------
# BASELINE.json configs at full size
# --------------------------------------------------------------------------

def test_config1_512_bit_exact():
    cfg = workloads.CONFIGS["1"]
    x = cfg.groups[0].image(0)
    st = check(x, cfg.levels, True, "config 1")
    assert st["max_abs_i"] == 0.0


def test_config2_4096_smooth():
    cfg = workloads.CONFIGS["2"]
    x = cfg.groups[0].image(0)
    st = check(x, cfg.levels, False, "config 2")
    assert st["max_abs_i"] <= 1e-4
    assert st["mismatch_ii"] == 0, st


@pytest.mark.parametrize("name", ["4", "4b"])
def test_config4_8level_smooth(name):
    cfg = workloads.CONFIGS[name]
    x = cfg.groups[0].image(0)
    st = check(x, cfg.levels, False, f"config {name}")
    assert st["max_abs_i"] <= 1e-4
    assert st["mismatch_ii"] == 0, st


def test_config3_16384_sampled():
    """Full 16384^2 image in the bench launch configuration; checked on every
    border quad of every subband plus 4 x 250k random positions with the
    pointwise brute-force convolution oracle (algorithm B), and everywhere
    with the exactness property (integer inputs -> every coefficient on the
    1/64 grid, |c| <= 1020)."""
    cfg = workloads.CONFIGS["3"]
    x = cfg.groups[0].image(0)
    H, W = x.shape
    got = gpu_forward(x, 1)
    rng = np.random.default_rng(3)
    b, m, n = sample_positions(W, H, 250_000, rng)
    ref = oracle.conv_sample(x, b, m, n)
    g = gather(got, W, H, b, m, n).astype(np.float64)
    np.testing.assert_array_equal(g, ref)
    scaled = got.astype(np.float64) * 64
    assert np.all(scaled == np.round(scaled))
    assert np.abs(got).max() <= 1020


def test_config3_16384_every_element():
    """Config 3 at full size, EVERY element of the Mallat output against the
    fp64 separable-lifting oracle (algorithm A) rounded to fp32 (oracle (ii)):
    bit for bit (integer inputs: the exact coefficient is representable).
    The oracle alone takes ~20 s and ~4.3 GB of host memory here."""
    cfg = workloads.CONFIGS["3"]
    x = cfg.groups[0].image(0)
    got = gpu_forward(x, 1)
    ref = oracle.forward(x.astype(np.float64), 1, round_f32=True)
    d = got.astype(np.float64) != ref
    assert not d.any(), f"{int(d.sum())} of {d.size} elements differ"


@pytest.mark.parametrize("W,H", [(16384, 8192), (20000, 6001), (20001, 6001)])
def test_large_level_tiles_sampled(W, H):
    """Levels large enough for the 15-row tile rule (tile_policy: >= 9 tiles
    per warp), incl. an odd height and a width that is not a slab multiple:
    border quads and 200k random positions against the pointwise oracle."""
    x = workloads.uniform_int(W, H, W + H)
    got = gpu_forward(x, 1)
    rng = np.random.default_rng(W)
    b, m, n = sample_positions(W, H, 200_000, rng)
    np.testing.assert_array_equal(gather(got, W, H, b, m, n).astype(np.float64), oracle.conv_sample(x, b, m, n))


def test_config5_batch_sampled():
    """Config 5 through dwt2_forward_batched (one launch per level over the
    group): 12 of each image size checked in full against the oracle (3
    levels; integer inputs -> exact at levels 1-2, oracle(ii) bit-exact at 3)."""
    cfg = workloads.CONFIGS["5"]
    for grp in cfg.groups:
        count = grp.count
        W, H = grp.width, grp.height
        xs = np.stack([grp.image(i) for i in range(count)])
        plan = dwt2.Plan(W, H, cfg.levels, max_count=count)
        out = plan.forward(torch.from_numpy(xs).cuda()).cpu().numpy()
        plan.close()
        for i in list(range(0, count, max(1, count // 12)))[:12]:
            x64 = xs[i].astype(np.float64)
            ref_ii = oracle.forward(x64, cfg.levels, round_f32=True)
            ref_i = oracle.forward(x64, cfg.levels, round_f32=False)
            st = compare(out[i], ref_i, ref_ii, False, f"config5 {W}x{H} #{i}")
            assert st["mismatch_ii"] == 0
            # levels 1-2 only (bottom/right parts written by levels 1, 2) are exact vs fp64
        # every image: batched == single-image path, bit for bit (sampled images)
        for i in (0, count - 1):
            np.testing.assert_array_equal(out[i], gpu_forward(xs[i], cfg.levels))


# --------------------------------------------------------------------------
# strips (the multi-GPU partition, emulated rank by rank on one GPU)
# --------------------------------------------------------------------------

def run_strips(x: np.ndarray, G: int, split_parts: bool) -> np.ndarray:
    """Transform x strip by strip with ghost rows copied from the full image,
    exactly the buffers each rank holds after the halo exchange, and
    assemble the global Mallat output."""
    from paper_1708_07853_b200 import distributed as dist_mod
    H, W = x.shape
    Hq = (H + 1) // 2
    full = np.empty_like(x)
    for g in range(G):
        r0, r1 = dist_mod.strip_rows(H, g, G)
        sp = dwt2.StripPlan(W, H, r0, r1)
        lo, hi = r0 - sp.ghost_top, r1 + sp.ghost_bot
        xin = torch.from_numpy(np.ascontiguousarray(x[lo:hi])).cuda()
        out = torch.full((r1 - r0, W), float("nan"), device="cuda")
        if split_parts:
            sp.forward(xin, out, dwt2.DWT2_STRIP_INTERIOR)
            sp.forward(xin, out, dwt2.DWT2_STRIP_BOUNDARY)
        else:
            sp.forward(xin, out, dwt2.DWT2_STRIP_ALL)
        o = out.cpu().numpy()
        sp.close()
        dist_mod.place_strip_output(full, o, W, H, r0, r1)
    return full


@pytest.mark.parametrize("W,H,G", [(1000, 777, 2), (1024, 1024, 3), (515, 260, 4), (2048, 2048, 8), (300, 33, 8)])
@pytest.mark.parametrize("split", [False, True])
def test_strips_equal_single_gpu(W, H, G, split):
    x = workloads.uniform_real(W, H, W + H + G)
    ref = gpu_forward(x, 1)
    got = run_strips(x, G, split)
    np.testing.assert_array_equal(got, ref)


def test_config3_strips_g8_bit_identical():
    """Config 3 at full size: the 8-strip decomposition (interior + boundary
    launches, as bench.py runs it per rank) equals the 1-GPU result bit for bit."""
    x = workloads.CONFIGS["3"].groups[0].image(0)
    ref = gpu_forward(x, 1)
    got = run_strips(x, 8, True)
    np.testing.assert_array_equal(got, ref)


# --------------------------------------------------------------------------
# API behaviour
# --------------------------------------------------------------------------

def test_host_entry_equals_device():
    for W, H, L in [(4096, 2048, 1), (1030, 777, 3), (8192, 8192, 8), (8193, 4099, 5), (5, 2000, 2)]:
        x = workloads.uniform_real(W, H, 9)
        ref = gpu_forward(x, L)
        plan = dwt2.Plan(W, H, L)
        hin = torch.from_numpy(x).pin_memory()
        hout = torch.empty_like(hin).pin_memory()
        plan.forward_host(hin, hout)
        plan.close()
        np.testing.assert_array_equal(hout.numpy(), ref)


def test_errors():
    with pytest.raises(dwt2.DWT2Error) as e:
        dwt2.Plan(1, 5, 1)
    assert e.value.code == dwt2.DWT2_EINVAL
    with pytest.raises(dwt2.DWT2Error) as e:
        dwt2.Plan(8, 8, 4)            # level 4 input would be 1x1
    assert e.value.code == dwt2.DWT2_EINVAL
    with pytest.raises(dwt2.DWT2Error) as e:
        dwt2.dwt2_plan_create(64, 64, 1, 7)
    assert e.value.code == dwt2.DWT2_EUNSUPPORTED
    plan = dwt2.Plan(64, 64, 1)
    x = torch.zeros(2 * 64 * 64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    with pytest.raises(dwt2.DWT2Error):       # overlapping in/out
        dwt2.dwt2_forward(plan.handle, x.data_ptr(), x.data_ptr() + 4 * 100, s)
    with pytest.raises(dwt2.DWT2Error):       # host pointer
        h = torch.zeros(64 * 64)
        dwt2.dwt2_forward(plan.handle, h.data_ptr(), x.data_ptr(), s)
    with pytest.raises(dwt2.DWT2Error):
        dwt2.dwt2_forward(plan.handle, 0, x.data_ptr(), s)
    info = plan.info()
    assert info.launches_per_forward == 1 and info.algorithmic_bytes == 8 * 64 * 64
    plan.close()


def test_negative_control_checker_flags_one_ulp():
    """The comparison used above must catch a single 1-ulp error anywhere."""
    x = workloads.uniform_real(130, 66, 4)
    got = gpu_forward(x, 2)
    ref_ii = oracle.forward(x.astype(np.float64), 2, round_f32=True)
    compare(got, None, ref_ii, True, "clean")
    for (r, c) in [(0, 0), (65, 129), (20, 100), (40, 3)]:
        bad = got.copy()
        bad[r, c] = np.nextafter(bad[r, c], np.float32(np.inf))
        with pytest.raises(AssertionError):
            compare(bad, None, ref_ii, True, "perturbed")
    assert ulp32(np.array([1.0]))[0] > 0


def test_errors_extended_api():
    """Argument checks of the entry points added for the 8f rows: strip
    levels, batched inverse, schemes, lifting plans; a failing call sets
    dwt2_last_error and a good call clears it."""
    s = torch.cuda.current_stream().cuda_stream
    lib = dwt2.lib()
    # strip level: bad level index, missing ll_out for a non-last level, part out of range
    sp = dwt2.StripPlan(64, 256, 0, 128, 2)
    buf = torch.zeros(129, 64, device="cuda")
    out = torch.zeros(128, 64, device="cuda")
    ll = torch.zeros(70, 32, device="cuda")
    for args in [(5, buf.data_ptr(), 64, ll.data_ptr(), 32, out.data_ptr(), 0),     # level 5 of a 2-level plan
                 (0, buf.data_ptr(), 64, 0, 0, out.data_ptr(), 0),                  # level 0 needs ll_out
                 (0, buf.data_ptr(), 64, ll.data_ptr(), 32, out.data_ptr(), 3),     # part 3
                 (0, buf.data_ptr(), 32, ll.data_ptr(), 32, out.data_ptr(), 0)]:    # in_pitch < width
        with pytest.raises(dwt2.DWT2Error):
            dwt2.dwt2_forward_strip_level(sp.handle, *args[:6], args[6], s)
        assert lib.dwt2_last_error() == dwt2.DWT2_EINVAL
    with pytest.raises(dwt2.DWT2Error):          # the one-level entry point on a 2-level strip plan
        dwt2.dwt2_forward_strip(sp.handle, buf.data_ptr(), out.data_ptr(), 0, s)
    sp.close()
    # batched inverse / scheme: count above the plan's max_count, unknown scheme
    plan = dwt2.Plan(64, 64, 1, max_count=2)
    a = torch.zeros(3, 64, 64, device="cuda")
    b = torch.zeros(3, 64, 64, device="cuda")
    with pytest.raises(dwt2.DWT2Error):
        dwt2.dwt2_inverse_batched(plan.handle, a.data_ptr(), b.data_ptr(), 3, 4096, 4096, s)
    with pytest.raises(dwt2.DWT2Error):
        dwt2.dwt2_forward_scheme(plan.handle, 42, a.data_ptr(), b.data_ptr(), 1, 4096, 4096, s)
    dwt2.dwt2_forward_scheme(plan.handle, dwt2.SCHEMES["sep_lifting"], a.data_ptr(), b.data_ptr(), 2, 4096, 4096, s)
    assert lib.dwt2_last_error() == dwt2.DWT2_OK
    plan.close()
    # wavelet plans: out-of-range wavelet id; strip plans are 5/3 only by construction
    with pytest.raises(dwt2.DWT2Error):
        dwt2.dwt2_plan_create_ex(64, 64, 1, 0, 9, 1)
    with pytest.raises(dwt2.DWT2Error) as e:
        dwt2.Plan(64, 64, 1, wavelet="cdf97").forward_host(torch.zeros(64, 64).pin_memory(),
                                                           torch.zeros(64, 64).pin_memory())
    assert e.value.code == dwt2.DWT2_EUNSUPPORTED


def test_determinism_across_runs_and_queue_orders():
    """Pin-10: the tile queues hand tiles out in a different
    order every run, yet every coefficient depends only on its own input
    neighbourhood, so repeated runs -- forward, inverse, 9/7, a batch and a
    mid-size (guided-tile) level -- are bit-identical."""
    cases = [(8192, 4096, 1, "cdf53", 1), (4096, 4096, 3, "cdf53", 1), (2048, 2048, 2, "cdf53", 6),
             (8192, 2048, 2, "cdf97", 1)]
    for W, H, L, wv, n in cases:
        x = torch.from_numpy(np.stack([workloads.uniform_real(W, H, 31 + i) for i in range(n)])).cuda()
        x = x[0] if n == 1 else x
        plan = dwt2.Plan(W, H, L, max_count=n, wavelet=wv)
        y0 = plan.forward(x).clone()
        r0 = plan.inverse(y0).clone()
        for _ in range(3):
            assert torch.equal(plan.forward(x), y0), (W, H, L, wv)
            assert torch.equal(plan.inverse(y0), r0), (W, H, L, wv)
        plan.close()
