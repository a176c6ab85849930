"""ctypes loader for the CPU oracle (oracle/dwt53_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product
package ``paper_1708_07853_b200``.  See the header of dwt53_oracle.c for what
each function computes and which PAPER.md passage it follows.

The shared library is compiled with plain ``gcc -O2 -ffp-contract=off`` (no
fused multiply-add contraction, no fast-math) by :func:`build` -- called by
``__graft_entry__.build()`` and lazily on first use.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "dwt53_oracle.c")
_SRCS = [_SRC, os.path.join(_HERE, "dwt97_oracle.c")]
_LIB = os.path.join(_HERE, "liboracle_dwt53.so")
_lib = None

BANDS = {"LL": 0, "HL": 1, "LH": 2, "HH": 3}


def build(force: bool = False) -> str:
    """Compile the oracle shared library (idempotent)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(os.path.getmtime(f) for f in _SRCS):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-Wall",
             "-shared", "-fPIC", *_SRCS, "-o", tmp])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        dp = ctypes.POINTER(ctypes.c_double)
        fp = ctypes.POINTER(ctypes.c_float)
        ip = ctypes.POINTER(ctypes.c_int)
        lp = ctypes.POINTER(ctypes.c_long)
        L = ctypes.c_long
        lib.oracle_dwt53_fwd_1d.argtypes = [dp, L, dp]
        lib.oracle_dwt53_inv_1d.argtypes = [dp, L, dp]
        lib.oracle_dwt53_fwd_lifting.argtypes = [dp, dp, L, L, L, ctypes.c_int]
        lib.oracle_dwt53_fwd_lifting.restype = L
        lib.oracle_dwt53_fwd_conv.argtypes = [dp, dp, L, L, L, ctypes.c_int]
        lib.oracle_dwt53_fwd_conv.restype = L
        lib.oracle_dwt53_inv_lifting.argtypes = [dp, dp, L, L, L, ctypes.c_int]
        lib.oracle_dwt53_inv_lifting.restype = L
        lib.oracle_dwt53_conv_sample_f32.argtypes = [fp, L, L, L, L, ip, lp, lp, dp]
        lib.oracle_dwt53_conv_sample.argtypes = [dp, L, L, L, L, ip, lp, lp, dp]
        lib.oracle_dwt97_fwd_1d.argtypes = [dp, L, dp]
        lib.oracle_dwt97_inv_1d.argtypes = [dp, L, dp]
        lib.oracle_dwt97_forward.argtypes = [dp, dp, L, L, L, ctypes.c_int, ctypes.c_int]
        lib.oracle_dwt97_forward.restype = L
        lib.oracle_dwt97_inverse.argtypes = [dp, dp, L, L, L, ctypes.c_int]
        lib.oracle_dwt97_inverse.restype = L
        lib.oracle_lift2_forward.argtypes = [dp, dp, L, L, L, ctypes.c_int, dp, ctypes.c_double]
        lib.oracle_lift2_forward.restype = L
        lib.oracle_dwt97_conv_sample_f32.argtypes = [fp, L, L, L, L, ip, lp, lp, dp]
        lib.oracle_wss_index.argtypes = [L, L]
        lib.oracle_wss_index.restype = L
        _lib = lib
    return _lib


def _dptr(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def fwd_1d(x) -> np.ndarray:
    """1-D forward lifting: [L (ceil(n/2)), H (floor(n/2))]."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _load().oracle_dwt53_fwd_1d(_dptr(x), x.size, _dptr(out))
    return out


def inv_1d(c) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.float64)
    out = np.empty_like(c)
    _load().oracle_dwt53_inv_1d(_dptr(c), c.size, _dptr(out))
    return out


def fwd_1d_97(x) -> np.ndarray:
    """1-D forward CDF 9/7 lifting: [low (ceil(n/2)), high (floor(n/2))]."""
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.empty_like(x)
    _load().oracle_dwt97_fwd_1d(_dptr(x), x.size, _dptr(out))
    return out


def inv_1d_97(c) -> np.ndarray:
    c = np.ascontiguousarray(c, dtype=np.float64)
    out = np.empty_like(c)
    _load().oracle_dwt97_inv_1d(_dptr(c), c.size, _dptr(out))
    return out


def forward(img, levels: int = 1, round_f32: bool = False, algorithm: str = "lifting",
            wavelet: str = "cdf53") -> np.ndarray:
    """Multi-level forward 2-D DWT of a H x W image, Mallat pyramid, fp64.

    wavelet: "cdf53" (dwt53_oracle.c) or "cdf97" (dwt97_oracle.c).
    algorithm: "lifting" (A, separable lifting) or "conv" (B, brute force).
    round_f32: round every level's output to fp32 before the next level
    (oracle output (ii) in DESIGN.md; False gives output (i)).
    """
    img = np.ascontiguousarray(img, dtype=np.float64)
    H, W = img.shape
    out = np.empty_like(img)
    if wavelet == "cdf97":
        r = _load().oracle_dwt97_forward(_dptr(img), _dptr(out), W, H, levels, int(bool(round_f32)),
                                         int(algorithm == "conv"))
    else:
        fn = _load().oracle_dwt53_fwd_lifting if algorithm == "lifting" else _load().oracle_dwt53_fwd_conv
        r = fn(_dptr(img), _dptr(out), W, H, levels, int(bool(round_f32)))
    if r < 0:
        raise ValueError("oracle: invalid arguments")
    return out


def forward_lifting2(img, levels: int, coeffs, K: float, round_f32: bool = False) -> np.ndarray:
    """General K <= 2 lifting wavelet: coeffs = (p1, u1, p2, u2), scaling K
    (low / K, high * K).  (-1/2, 1/4, 0, 0), 1 is CDF 5/3; the 9/7 constants
    give CDF 9/7 (both pinned in the tests)."""
    img = np.ascontiguousarray(img, dtype=np.float64)
    H, W = img.shape
    out = np.empty_like(img)
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    assert c.size == 4
    if _load().oracle_lift2_forward(_dptr(img), _dptr(out), W, H, levels, int(bool(round_f32)), _dptr(c),
                                    float(K)) < 0:
        raise ValueError("oracle: invalid arguments")
    return out


def inverse(coeffs, levels: int = 1, round_f32: bool = False, wavelet: str = "cdf53") -> np.ndarray:
    """Multi-level inverse (algorithm C) of a Mallat pyramid, fp64.
    round_f32: round every level's reconstruction to fp32 (the GPU storage type)."""
    c = np.ascontiguousarray(coeffs, dtype=np.float64)
    H, W = c.shape
    out = np.empty_like(c)
    fn = _load().oracle_dwt97_inverse if wavelet == "cdf97" else _load().oracle_dwt53_inv_lifting
    if fn(_dptr(c), _dptr(out), W, H, levels, int(bool(round_f32))) < 0:
        raise ValueError("oracle: invalid arguments")
    return out


def conv_sample(img, band, m, n, wavelet: str = "cdf53") -> np.ndarray:
    """Pointwise brute-force convolution (algorithm B) of one level.

    img: H x W array (fp32 or fp64; rows may have a pitch >= W via a 2-D view
    with unit column stride).  band/m/n: equal-length integer arrays.
    """
    band = np.ascontiguousarray(band, dtype=np.int32)
    m = np.ascontiguousarray(m, dtype=np.int64)
    n = np.ascontiguousarray(n, dtype=np.int64)
    assert band.shape == m.shape == n.shape
    H, W = img.shape
    assert img.strides[1] == img.itemsize
    pitch = img.strides[0] // img.itemsize
    res = np.empty(band.size, dtype=np.float64)
    lib = _load()
    ip = band.ctypes.data_as(ctypes.POINTER(ctypes.c_int))
    mp = m.ctypes.data_as(ctypes.POINTER(ctypes.c_long))
    nq = n.ctypes.data_as(ctypes.POINTER(ctypes.c_long))
    if wavelet == "cdf97":
        if img.dtype != np.float32:
            raise TypeError("cdf97 samples: fp32 images")
        lib.oracle_dwt97_conv_sample_f32(img.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                         pitch, W, H, band.size, ip, mp, nq, _dptr(res))
    elif img.dtype == np.float32:
        lib.oracle_dwt53_conv_sample_f32(img.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                         pitch, W, H, band.size, ip, mp, nq, _dptr(res))
    elif img.dtype == np.float64:
        lib.oracle_dwt53_conv_sample(_dptr(img), pitch, W, H, band.size, ip, mp, nq, _dptr(res))
    else:
        raise TypeError(img.dtype)
    return res


def wss_index(k: int, n: int) -> int:
    return int(_load().oracle_wss_index(k, n))


def level_dims(W: int, H: int, levels: int):
    """[(W_k, H_k)] input size of every level: W_{k+1} = ceil(W_k / 2)."""
    dims = []
    w, h = W, H
    for _ in range(levels):
        dims.append((w, h))
        w, h = (w + 1) // 2, (h + 1) // 2
    return dims
