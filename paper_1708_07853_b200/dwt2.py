"""Thin Python binding of the C ABI in include/dwt2.h (argument marshalling only).

Every function here forwards to libdwt2.so; every step of the transform runs
in the CUDA kernels behind it.  There is no CPU fallback: if the library is
missing or cannot be loaded, import-time use raises ``RuntimeError``.

torch is used only for device memory and streams (tensors' data pointers and
``torch.cuda.current_stream().cuda_stream``), as BASELINE.json north_star says.
"""
from __future__ import annotations

import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libdwt2.so")      # the in-tree product library (no environment override)

DWT2_OK, DWT2_EINVAL, DWT2_ENOMEM, DWT2_ECUDA, DWT2_EUNSUPPORTED, DWT2_ETIMEOUT = 0, -1, -2, -3, -4, -5
DWT2_PEER_RANKS, DWT2_PEER_SEQUENTIAL = 0, 1
DWT2_BOUNDARY_SYMMETRIC = 0
DWT2_STRIP_ALL, DWT2_STRIP_INTERIOR, DWT2_STRIP_BOUNDARY, DWT2_STRIP_PUBLISH = 0, 1, 2, 3
DWT2_WAVELET_CDF53, DWT2_WAVELET_CDF97, DWT2_WAVELET_CDF53_K2, DWT2_WAVELET_LIFTING = 0, 1, 2, 3
WAVELETS = {"cdf53": 0, "cdf97": 1, "cdf53_k2": 2, "lifting": 3}
SCHEMES = {"fused": 0, "nonsep_naive": 1, "nonsep_lifting": 2, "nonsep_adapted": 3, "sep_conv": 4,
           "sep_lifting": 5, "fused_literal": 6, "fused_adapted": 7}

# symbol -> (restype, argtypes); mirrors include/dwt2.h exactly
_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64


class StripLevel(ctypes.Structure):
    _fields_ = [("width", _I32), ("global_height", _I32), ("row_begin", _I32), ("row_end", _I32),
                ("ghost_top", _I32), ("ghost_bot", _I32)]


class PlanInfo(ctypes.Structure):
    _fields_ = [("width", _I32), ("height", _I32), ("levels", _I32), ("max_count", _I32),
                ("launches_per_forward", _I32), ("tma_levels", _I32),
                ("algorithmic_bytes", _I64), ("scratch_bytes", _I64)]


class PeerDesc(ctypes.Structure):
    """dwt2_peer_desc_t: what a neighbour needs to map a peer strip context."""
    _fields_ = [("ipc_handle", ctypes.c_uint8 * 64), ("base", ctypes.c_uint64), ("pid", _I64),
                ("device", _I32), ("width", _I32), ("global_height", _I32), ("levels", _I32),
                ("row_begin", _I32), ("row_end", _I32), ("timeout_ms", _I32), ("reserved", _I32),
                ("owned_off", _I64 * 32), ("pitch", _I64 * 32), ("flags_off", _I64)]

    def to_bytes(self) -> bytes:
        return bytes(self)

    @classmethod
    def from_bytes(cls, b: bytes) -> "PeerDesc":
        if len(b) != ctypes.sizeof(cls):
            raise ValueError(f"peer descriptor: {len(b)} bytes, expected {ctypes.sizeof(cls)}")
        return cls.from_buffer_copy(b)


SIGNATURES = {
    "dwt2_plan_create": (_P, [_I32, _I32, _I32, _I32]),
    "dwt2_plan_create_batched": (_P, [_I32, _I32, _I32, _I32, _I32]),
    "dwt2_plan_create_ex": (_P, [_I32, _I32, _I32, _I32, _I32, _I32]),
    "dwt2_plan_create_lifting": (_P, [_I32, _I32, _I32, _I32, ctypes.POINTER(ctypes.c_double), ctypes.c_double, _I32]),
    "dwt2_plan_create_strip": (_P, [_I32, _I32, _I32, _I32, _I32]),
    "dwt2_plan_create_strip_levels": (_P, [_I32, _I32, _I32, _I32, _I32, _I32]),
    "dwt2_strip_level_info": (_I32, [_P, _I32, ctypes.POINTER(StripLevel)]),
    "dwt2_forward_strip_level": (_I32, [_P, _I32, _P, _I64, _P, _I64, _P, _I32, _P]),
    "dwt2_forward": (_I32, [_P, _P, _P, _P]),
    "dwt2_forward_batched": (_I32, [_P, _P, _P, _I32, _I64, _I64, _P]),
    "dwt2_forward_strip": (_I32, [_P, _P, _P, _I32, _P]),
    "dwt2_forward_host": (_I32, [_P, _P, _P, _P]),
    "dwt2_peer_strip_create": (_P, [_P, _I32]),
    "dwt2_peer_strip_buffer": (_I32, [_P, _I32, ctypes.POINTER(_P), ctypes.POINTER(_I64)]),
    "dwt2_peer_strip_export": (_I32, [_P, ctypes.POINTER(PeerDesc)]),
    "dwt2_peer_strip_connect": (_I32, [_P, ctypes.POINTER(PeerDesc), ctypes.POINTER(PeerDesc), _I32]),
    "dwt2_peer_strip_level": (_I32, [_P, _I32, _I32, _P, _P]),
    "dwt2_peer_strip_forward": (_I32, [_P, _P, _P]),
    "dwt2_peer_strip_status": (_I32, [_P]),
    "dwt2_peer_strip_destroy": (None, [_P]),
    "dwt2_inverse": (_I32, [_P, _P, _P, _P]),
    "dwt2_inverse_batched": (_I32, [_P, _P, _P, _I32, _I64, _I64, _P]),
    "dwt2_scheme_steps": (_I32, [_I32]),
    "dwt2_forward_scheme": (_I32, [_P, _I32, _P, _P, _I32, _I64, _I64, _P]),
    "dwt2_destroy": (None, [_P]),
    "dwt2_plan_info": (_I32, [_P, ctypes.POINTER(PlanInfo)]),
    "dwt2_last_error": (_I32, []),
    "dwt2_error_string": (ctypes.c_char_p, [_I32]),
    "dwt2_version": (ctypes.c_char_p, []),
}

_lib = None


class DWT2Error(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {error_string(code)} ({code})")


def use_variant(path: str) -> None:
    """Measurement scripts only: load a tuning build (build/variants/, see
    _build.build_variant) instead of the product library.  Must be called
    before the first call into the library."""
    global LIB_PATH
    if _lib is not None:
        raise RuntimeError("libdwt2 is already loaded")
    LIB_PATH = os.path.abspath(path)


def lib() -> ctypes.CDLL:
    """Load libdwt2.so (in-tree).  Raises if it is absent: no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                               "(nvcc for sm_100a); there is no CPU fallback")
        l = ctypes.CDLL(LIB_PATH)
        product = os.path.abspath(LIB_PATH) == os.path.join(_PKG, "libdwt2.so")
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(l, name, None)
            if fn is None:
                if product:
                    raise RuntimeError(f"{LIB_PATH} does not export {name}: rebuild (__graft_entry__.build())")
                continue                  # an older measurement build (use_variant) without this entry point
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def error_string(code: int) -> str:
    return lib().dwt2_error_string(code).decode()


def version() -> str:
    return lib().dwt2_version().decode()


def _check(code: int, what: str) -> None:
    if code != DWT2_OK:
        raise DWT2Error(code, what)


def _plan_or_raise(ptr, what):
    if not ptr:
        raise DWT2Error(lib().dwt2_last_error(), what)
    return ptr


# ---- raw C-ABI names (pointers are ints) -------------------------------------

def dwt2_plan_create(width, height, levels, boundary=DWT2_BOUNDARY_SYMMETRIC):
    return _plan_or_raise(lib().dwt2_plan_create(width, height, levels, boundary), "dwt2_plan_create")


def dwt2_plan_create_batched(width, height, levels, boundary, max_count):
    return _plan_or_raise(lib().dwt2_plan_create_batched(width, height, levels, boundary, max_count),
                          "dwt2_plan_create_batched")


def dwt2_plan_create_ex(width, height, levels, boundary, wavelet, max_count):
    return _plan_or_raise(lib().dwt2_plan_create_ex(width, height, levels, boundary, wavelet, max_count),
                          "dwt2_plan_create_ex")


def dwt2_plan_create_lifting(width, height, levels, boundary, coeffs, K, max_count):
    c = (ctypes.c_double * 4)(*[float(v) for v in coeffs])
    return _plan_or_raise(lib().dwt2_plan_create_lifting(width, height, levels, boundary, c, float(K), max_count),
                          "dwt2_plan_create_lifting")


def dwt2_plan_create_strip(width, global_height, row_begin, row_end, boundary=DWT2_BOUNDARY_SYMMETRIC):
    return _plan_or_raise(lib().dwt2_plan_create_strip(width, global_height, row_begin, row_end, boundary),
                          "dwt2_plan_create_strip")


def dwt2_plan_create_strip_levels(width, global_height, row_begin, row_end, levels,
                                  boundary=DWT2_BOUNDARY_SYMMETRIC):
    return _plan_or_raise(lib().dwt2_plan_create_strip_levels(width, global_height, row_begin, row_end, levels,
                                                              boundary), "dwt2_plan_create_strip_levels")


def dwt2_strip_level_info(plan, level) -> StripLevel:
    info = StripLevel()
    _check(lib().dwt2_strip_level_info(plan, level, ctypes.byref(info)), "dwt2_strip_level_info")
    return info


def dwt2_forward_strip_level(plan, level, in_ptr, in_pitch, ll_ptr, ll_pitch, out_ptr, part, stream):
    _check(lib().dwt2_forward_strip_level(plan, level, in_ptr, in_pitch, ll_ptr, ll_pitch, out_ptr, part, stream),
           "dwt2_forward_strip_level")


def dwt2_forward(plan, in_ptr, out_ptr, stream):
    _check(lib().dwt2_forward(plan, in_ptr, out_ptr, stream), "dwt2_forward")


def dwt2_forward_batched(plan, in_ptr, out_ptr, count, in_stride, out_stride, stream):
    _check(lib().dwt2_forward_batched(plan, in_ptr, out_ptr, count, in_stride, out_stride, stream),
           "dwt2_forward_batched")


def dwt2_forward_strip(plan, in_ptr, out_ptr, part, stream):
    _check(lib().dwt2_forward_strip(plan, in_ptr, out_ptr, part, stream), "dwt2_forward_strip")


def dwt2_forward_host(plan, host_in_ptr, host_out_ptr, stream):
    _check(lib().dwt2_forward_host(plan, host_in_ptr, host_out_ptr, stream), "dwt2_forward_host")


def dwt2_peer_strip_create(plan, timeout_ms=0):
    return _plan_or_raise(lib().dwt2_peer_strip_create(plan, timeout_ms), "dwt2_peer_strip_create")


def dwt2_peer_strip_buffer(ctx, level):
    """(device pointer of level's first owned row, row pitch in floats)"""
    ptr, pitch = _P(), _I64()
    _check(lib().dwt2_peer_strip_buffer(ctx, level, ctypes.byref(ptr), ctypes.byref(pitch)),
           "dwt2_peer_strip_buffer")
    return ptr.value, pitch.value


def dwt2_peer_strip_export(ctx) -> PeerDesc:
    d = PeerDesc()
    _check(lib().dwt2_peer_strip_export(ctx, ctypes.byref(d)), "dwt2_peer_strip_export")
    return d


def dwt2_peer_strip_connect(ctx, above, below, mode):
    _check(lib().dwt2_peer_strip_connect(ctx, None if above is None else ctypes.byref(above),
                                         None if below is None else ctypes.byref(below), mode),
           "dwt2_peer_strip_connect")


def dwt2_peer_strip_level(ctx, level, part, out_ptr, stream):
    _check(lib().dwt2_peer_strip_level(ctx, level, part, out_ptr, stream), "dwt2_peer_strip_level")


def dwt2_peer_strip_forward(ctx, out_ptr, stream):
    _check(lib().dwt2_peer_strip_forward(ctx, out_ptr, stream), "dwt2_peer_strip_forward")


def dwt2_peer_strip_status(ctx):
    return lib().dwt2_peer_strip_status(ctx)


def dwt2_peer_strip_destroy(ctx):
    lib().dwt2_peer_strip_destroy(ctx)


def dwt2_inverse(plan, in_ptr, out_ptr, stream):
    _check(lib().dwt2_inverse(plan, in_ptr, out_ptr, stream), "dwt2_inverse")


def dwt2_inverse_batched(plan, in_ptr, out_ptr, count, in_stride, out_stride, stream):
    _check(lib().dwt2_inverse_batched(plan, in_ptr, out_ptr, count, in_stride, out_stride, stream),
           "dwt2_inverse_batched")


def dwt2_scheme_steps(scheme):
    r = lib().dwt2_scheme_steps(scheme)
    if r < 0:
        raise DWT2Error(r, "dwt2_scheme_steps")
    return r


def dwt2_forward_scheme(plan, scheme, in_ptr, out_ptr, count, in_stride, out_stride, stream):
    _check(lib().dwt2_forward_scheme(plan, scheme, in_ptr, out_ptr, count, in_stride, out_stride, stream),
           "dwt2_forward_scheme")


def dwt2_destroy(plan):
    lib().dwt2_destroy(plan)


def dwt2_plan_info(plan) -> PlanInfo:
    info = PlanInfo()
    _check(lib().dwt2_plan_info(plan, ctypes.byref(info)), "dwt2_plan_info")
    return info


# ---- torch-facing convenience (marshalling only) ------------------------------

def _stream_handle(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _check_image(x, name):
    import torch
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32 or not x.is_contiguous():
        raise ValueError(f"{name} must be a contiguous float32 CUDA tensor")


class Plan:
    """Owns a dwt2_plan* (see include/dwt2.h)."""

    def __init__(self, width: int, height: int, levels: int = 1, max_count: int = 1, wavelet: str = "cdf53",
                 lifting=None):
        """wavelet: "cdf53" (product 5/3 kernel), "cdf97", "cdf53_k2" or
        "lifting" with lifting = (p1, u1, p2, u2, K)."""
        self.width, self.height, self.levels, self.max_count = width, height, levels, max_count
        self.wavelet = wavelet
        if wavelet == "lifting":
            p1, u1, p2, u2, K = lifting
            self._p = dwt2_plan_create_lifting(width, height, levels, DWT2_BOUNDARY_SYMMETRIC, (p1, u1, p2, u2), K,
                                               max_count)
        elif wavelet != "cdf53":
            self._p = dwt2_plan_create_ex(width, height, levels, DWT2_BOUNDARY_SYMMETRIC, WAVELETS[wavelet],
                                          max_count)
        elif max_count == 1:
            self._p = dwt2_plan_create(width, height, levels)
        else:
            self._p = dwt2_plan_create_batched(width, height, levels, DWT2_BOUNDARY_SYMMETRIC, max_count)

    @property
    def handle(self):
        return self._p

    def info(self) -> PlanInfo:
        return dwt2_plan_info(self._p)

    def forward(self, x, out=None, stream=None):
        _check_image(x, "x")
        if tuple(x.shape[-2:]) != (self.height, self.width):
            raise ValueError(f"expected (..., {self.height}, {self.width}), got {tuple(x.shape)}")
        import torch
        if out is None:
            out = torch.empty_like(x)
        _check_image(out, "out")
        if x.dim() == 2:
            dwt2_forward(self._p, x.data_ptr(), out.data_ptr(), _stream_handle(stream))
        else:
            n = x.numel() // (self.width * self.height)
            img = self.width * self.height
            dwt2_forward_batched(self._p, x.data_ptr(), out.data_ptr(), n, img, img, _stream_handle(stream))
        return out

    def forward_scheme(self, scheme, x, out=None, stream=None):
        """Forward transform with one of the paper's schemes (SCHEMES), one
        kernel per step; scheme "fused" is forward()."""
        _check_image(x, "x")
        if tuple(x.shape[-2:]) != (self.height, self.width):
            raise ValueError(f"expected (..., {self.height}, {self.width}), got {tuple(x.shape)}")
        import torch
        if out is None:
            out = torch.empty_like(x)
        _check_image(out, "out")
        img = self.width * self.height
        n = x.numel() // img
        code = SCHEMES[scheme] if isinstance(scheme, str) else int(scheme)
        dwt2_forward_scheme(self._p, code, x.data_ptr(), out.data_ptr(), n, img, img, _stream_handle(stream))
        return out

    def inverse(self, y, out=None, stream=None):
        """Reconstruct (H, W) or (N, H, W) images from their Mallat pyramids."""
        _check_image(y, "y")
        if tuple(y.shape[-2:]) != (self.height, self.width):
            raise ValueError(f"expected (..., {self.height}, {self.width}), got {tuple(y.shape)}")
        import torch
        if out is None:
            out = torch.empty_like(y)
        _check_image(out, "out")
        if y.dim() == 2:
            dwt2_inverse(self._p, y.data_ptr(), out.data_ptr(), _stream_handle(stream))
        else:
            n = y.numel() // (self.width * self.height)
            img = self.width * self.height
            dwt2_inverse_batched(self._p, y.data_ptr(), out.data_ptr(), n, img, img, _stream_handle(stream))
        return out

    def forward_host(self, host_in, host_out, stream=None):
        """host_in / host_out: CPU float32 contiguous H x W tensors (pinned for
        full speed).  Checked here because the C call copies W*H floats from
        and to the raw host pointers."""
        import torch
        for name, t in (("host_in", host_in), ("host_out", host_out)):
            if not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != torch.float32 \
                    or not t.is_contiguous() or t.numel() != self.width * self.height:
                raise ValueError(f"{name}: need a contiguous CPU float32 tensor of {self.height} x {self.width} "
                                 f"elements")
        if self.max_count != 1:
            raise ValueError("forward_host: single-image plans only")
        dwt2_forward_host(self._p, host_in.data_ptr(), host_out.data_ptr(), _stream_handle(stream))
        return host_out

    def close(self):
        if getattr(self, "_p", None):
            dwt2_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class StripPlan:
    """Plan for the row strip [row_begin, row_end) of a W x Hg image, `levels`
    levels with one halo exchange per level (levels = 1: config 3)."""

    def __init__(self, width: int, global_height: int, row_begin: int, row_end: int, levels: int = 1):
        self.width, self.global_height, self.levels = width, global_height, levels
        self.row_begin, self.row_end = row_begin, row_end
        self._p = dwt2_plan_create_strip_levels(width, global_height, row_begin, row_end, levels)
        self.level_info = [dwt2_strip_level_info(self._p, k) for k in range(levels)]
        self.ghost_top = self.level_info[0].ghost_top
        self.ghost_bot = self.level_info[0].ghost_bot

    @property
    def handle(self):
        return self._p

    @property
    def in_rows(self) -> int:
        return self.row_end - self.row_begin + self.ghost_top + self.ghost_bot

    def forward(self, x_with_ghosts, out, part=DWT2_STRIP_ALL, stream=None):
        """One-level plans: level 0 from the ghost-padded strip (pitch W)."""
        _check_image(x_with_ghosts, "x")
        _check_image(out, "out")
        dwt2_forward_strip(self._p, x_with_ghosts.data_ptr(), out.data_ptr(), part, _stream_handle(stream))
        return out

    def forward_level(self, level, buf, ll_out, out, part=DWT2_STRIP_ALL, stream=None):
        """Level `level`: buf = its ghost-padded input (2-D tensor, row pitch =
        buf.stride(0)); ll_out = 2-D view of the next level's owned rows (None
        for the last level); out = the strip-local pyramid (W x rows)."""
        _check_image(out, "out")
        ll_ptr, ll_pitch = (0, 0) if ll_out is None else (ll_out.data_ptr(), ll_out.stride(0))
        dwt2_forward_strip_level(self._p, level, buf.data_ptr(), buf.stride(0), ll_ptr, ll_pitch, out.data_ptr(),
                                 part, _stream_handle(stream))
        return out

    def close(self):
        if getattr(self, "_p", None):
            dwt2_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _DeviceArray:
    """__cuda_array_interface__ of a float32 region the C library owns (torch.as_tensor wraps it)."""

    def __init__(self, ptr, rows, cols, pitch):
        self.__cuda_array_interface__ = {"shape": (rows, cols), "typestr": "<f4", "data": (ptr, False),
                                         "strides": (pitch * 4, 4), "version": 3}


class PeerStrip:
    """A peer strip context (include/dwt2.h): the rank's level buffers and
    flags in one device allocation; the halo of every level is read from the
    neighbours' contexts by the BOUNDARY kernels (no message exchange)."""

    def __init__(self, plan: StripPlan, timeout_ms: int = 0):
        self.plan = plan                      # the C context points at the plan: keep it alive
        self._c = dwt2_peer_strip_create(plan.handle, timeout_ms)

    @property
    def handle(self):
        return self._c

    def owned(self, level: int):
        """torch view of level's owned rows (level 0: write the strip's pixels here)."""
        import torch
        info = self.plan.level_info[level]
        ptr, pitch = dwt2_peer_strip_buffer(self._c, level)
        arr = _DeviceArray(ptr, info.row_end - info.row_begin, info.width, pitch)
        return torch.as_tensor(arr, device=torch.device("cuda", torch.cuda.current_device()))

    def export(self) -> PeerDesc:
        return dwt2_peer_strip_export(self._c)

    def connect(self, above, below, mode=DWT2_PEER_RANKS):
        dwt2_peer_strip_connect(self._c, above, below, mode)

    def level(self, level, part, out, stream=None):
        _check_image(out, "out")
        dwt2_peer_strip_level(self._c, level, part, out.data_ptr(), _stream_handle(stream))
        return out

    def forward(self, out, stream=None):
        _check_image(out, "out")
        dwt2_peer_strip_forward(self._c, out.data_ptr(), _stream_handle(stream))
        return out

    def status(self) -> int:
        return dwt2_peer_strip_status(self._c)

    def close(self):
        if getattr(self, "_c", None):
            dwt2_peer_strip_destroy(self._c)
            self._c = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def inverse(y, levels: int = 1):
    """One-shot inverse DWT of a (H, W) or (N, H, W) CUDA float32 Mallat pyramid."""
    p = Plan(y.shape[-1], y.shape[-2], levels, max_count=max(1, y.numel() // (y.shape[-1] * y.shape[-2])))
    try:
        return p.inverse(y)
    finally:
        import torch
        torch.cuda.current_stream().synchronize()
        p.close()


def forward(x, levels: int = 1):
    """One-shot forward DWT of a (H, W) or (N, H, W) CUDA float32 tensor."""
    p = Plan(x.shape[-1], x.shape[-2], levels, max_count=max(1, x.numel() // (x.shape[-1] * x.shape[-2])))
    try:
        return p.forward(x)
    finally:
        import torch
        torch.cuda.current_stream().synchronize()
        p.close()
