"""paper_1602_02740_b200 -- thin Python binding over libtoomgpu (C ABI in
include/toomgpu.h).  Argument marshalling only: every step of the Toom-Cook
path runs in the CUDA kernels of csrc/.  PyTorch supplies device memory and
streams.  There is no CPU fallback: if the library or a CUDA device is
missing, every call raises.

    import paper_1602_02740_b200 as tg
    w = tg.toom_mul_batched(u, v, B=4)              # u, v: [batch][n] uint32 CUDA tensors
    w = tg.toom_mul(u, v, B=4)                      # 1-D operands, w has nu+nv limbs
"""
from __future__ import annotations

import ctypes
import os

import torch

from .build import LIB

_lib = None

TOOM_OK, TOOM_EINVAL, TOOM_EVERIFY, TOOM_EINEXACT, TOOM_ENOMEM, TOOM_ECUDA, TOOM_EUNSUPPORTED = range(7)


class ToomError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {lib().toom_status_string(status).decode()} ({status})")
        self.status = status


class ToomPlan(ctypes.Structure):
    """toom_plan_t: top_B, t4, t3, chunk, long_count (see include/toomgpu.h)."""
    _fields_ = [("top_B", ctypes.c_int), ("t4", ctypes.c_size_t), ("t3", ctypes.c_size_t), ("chunk", ctypes.c_size_t),
                ("long_count", ctypes.c_size_t)]


def plan(B: int, t4: int = 256, t3: int = 64, chunk: int = 0, long_count: int = 0) -> ToomPlan:
    return ToomPlan(B, t4, t3, chunk, long_count)


# exported symbols and their ctypes signatures (tests check every symbol of
# include/toomgpu.h is here and exported by the .so)
_P = ctypes.c_void_p
_SZ = ctypes.c_size_t
_I = ctypes.c_int
SIGNATURES = {
    "toom_default_plan": (ToomPlan, [_I]),
    "toom_mul_batched": (_I, [_P, _P, _P, _SZ, _SZ, _I, _P]),
    "toom_mul_batched_plan": (_I, [_P, _P, _P, _SZ, _SZ, ctypes.POINTER(ToomPlan), _P]),
    "toom_mul": (_I, [_P, _P, _SZ, _P, _SZ, _I, _P]),
    "toom_mul_batched_host": (_I, [_P, _P, _P, _SZ, _SZ, ctypes.POINTER(ToomPlan), _P]),
    "toom_workspace_bytes": (_SZ, [_SZ, _SZ, ctypes.POINTER(ToomPlan)]),
    "toom_set_workspace": (_I, [_P, _SZ]),
    "toom_last_error": (_I, []),
    "toom_status_string": (ctypes.c_char_p, [_I]),
    "toom_last_launch_count": (_SZ, []),
    "toom_base_interleaved": (_I, [_P, _P, _P, _SZ, _SZ, _P]),
    "toom_base_interleaved_tc": (_I, [_P, _P, _P, _SZ, _SZ, _P]),
    "toom_eval_top": (_I, [_P, _P, _SZ, _SZ, _I, _P]),
    "toom_eval_width": (_SZ, [_SZ, _I]),
    "toom_npoints": (_I, [_I]),
    "toom_profile_enable": (None, [_I]),
    "toom_set_fused": (None, [_I]),
    "toom_set_top_stream": (None, [_I]),
    "toom_profile_collect": (_I, [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_size_t), _I]),
    "toom_plan_describe": (_SZ, [_SZ, _SZ, ctypes.POINTER(ToomPlan), ctypes.c_char_p, _SZ]),
    "toom_probe_limb_products": (ctypes.c_double, [ctypes.POINTER(ctypes.c_double), _P]),
    "toom_probe_carry_chain": (ctypes.c_double, [ctypes.POINTER(ctypes.c_double), _P]),
    "toom_eval_points": (_I, [_P, _P, _SZ, _SZ, _I, _I, _P]),
    "toom_eval_points_range": (_I, [_P, _P, _SZ, _SZ, _I, _I, _I, _I, _P]),
    "toom_interp_recompose": (_I, [_P, _P, _SZ, _SZ, _I, _P]),
    "toom_mul_signed_batched": (_I, [_P, _P, _P, _SZ, _SZ, ctypes.POINTER(ToomPlan), _P]),
    "toom_product_width_point": (_SZ, [_SZ, _I]),
    "toom_set_check": (None, [_I]),
    "toom_mul_ntt": (_I, [_P, _P, _SZ, _P, _SZ, _I, _P]),
    "toom_sqr_batched": (_I, [_P, _P, _SZ, _SZ, ctypes.POINTER(ToomPlan), _P]),
    "toom_set_t16_matrix": (None, [_I]),
    "toom_set_c2_mode": (None, [_I]),
    "toom_set_lazy_bottom": (None, [_I]),
    "toom_set_verify": (None, [_I]),
    "toom_debug_fault": (None, [_I]),
}


def lib():
    """Load libtoomgpu.so (built in-tree by build.py / __graft_entry__.build())."""
    global _lib
    if _lib is None:
        path = os.environ.get("TOOM_LIB") or LIB   # experiments: an alternative build of the same sources
        if not os.path.exists(path):
            raise RuntimeError(f"libtoomgpu.so not built ({path}); run python -m paper_1602_02740_b200.build")
        L = ctypes.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _check(st: int, what: str):
    if st != TOOM_OK:
        raise ToomError(st, what)


def _dev(t: torch.Tensor, name: str) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if t.element_size() != 4 or not t.is_contiguous():
        raise TypeError(f"{name} must be a contiguous 32-bit tensor")
    return t.data_ptr()


def _out(t: torch.Tensor, name: str, shape, like: torch.Tensor) -> int:
    """A caller-supplied output must have exactly the result's shape, dtype
    and device (the library writes every limb of it and nothing beyond)."""
    if tuple(t.shape) != tuple(shape) or t.dtype != like.dtype or t.device != like.device:
        raise ValueError(f"{name} must be a {like.dtype} tensor of shape {tuple(shape)} on {like.device}, "
                         f"got {t.dtype} {tuple(t.shape)} on {t.device}")
    return _dev(t, name)


def _stream(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def toom_mul_batched(u: torch.Tensor, v: torch.Tensor, B: int = 4, t4: int = 256, t3: int = 64, chunk: int = 0,
                     out: torch.Tensor | None = None, stream=None, long_count: int = 0) -> torch.Tensor:
    """w[i] = u[i] * v[i]; u, v: [batch][n] uint32 CUDA tensors; returns [batch][2n]."""
    if u.shape != v.shape or u.dim() != 2:
        raise ValueError("u and v must both be [batch][n]")
    batch, n = u.shape
    if out is None:
        out = torch.empty((batch, 2 * n), dtype=u.dtype, device=u.device)
    p = plan(B, t4, t3, chunk, long_count)
    st = lib().toom_mul_batched_plan(_out(out, "out", (batch, 2 * n), u), _dev(u, "u"), _dev(v, "v"), n, batch,
                                     ctypes.byref(p),
                                     _stream(stream))
    _check(st, "toom_mul_batched")
    return out


def toom_sqr_batched(u: torch.Tensor, B: int = 4, t4: int = 256, t3: int = 64, chunk: int = 0,
                     out: torch.Tensor | None = None, stream=None, long_count: int = 0) -> torch.Tensor:
    """w[i] = u[i]^2 (squaring specialisation); u: [batch][n] uint32 CUDA tensor."""
    if u.dim() != 2:
        raise ValueError("u must be [batch][n]")
    batch, n = u.shape
    if out is None:
        out = torch.empty((batch, 2 * n), dtype=u.dtype, device=u.device)
    p = plan(B, t4, t3, chunk, long_count)
    st = lib().toom_sqr_batched(_out(out, "out", (batch, 2 * n), u), _dev(u, "u"), n, batch, ctypes.byref(p),
                                _stream(stream))
    _check(st, "toom_sqr_batched")
    return out


def toom_mul(u: torch.Tensor, v: torch.Tensor, B: int = 4, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """w = u * v for 1-D uint32 CUDA tensors; returns nu+nv limbs."""
    nu, nv = u.numel(), v.numel()
    if out is None:
        out = torch.empty(nu + nv, dtype=u.dtype, device=u.device)
    if u.dim() != 1 or v.dim() != 1 or u.dtype != v.dtype:
        raise ValueError("u and v must be 1-D tensors of one dtype")
    st = lib().toom_mul(_out(out, "out", (nu + nv,), u), _dev(u, "u") if nu else None, nu, _dev(v, "v") if nv else None, nv, B,
                        _stream(stream))
    _check(st, "toom_mul")
    return out


def toom_mul_batched_host(u, v, B: int = 4, t4: int = 256, t3: int = 64, chunk: int = 0, out=None, stream=None):
    """End-to-end call with HOST buffers (torch CPU tensors or numpy arrays,
    pinned ideally): H2D copies, multiply, D2H copy, stream sync -- all in C."""
    import numpy as np

    def ptr(x):
        if isinstance(x, torch.Tensor):
            assert not x.is_cuda and x.is_contiguous() and x.element_size() == 4
            return x.data_ptr()
        assert isinstance(x, np.ndarray) and x.dtype == np.uint32 and x.flags.c_contiguous
        return x.ctypes.data

    batch, n = u.shape
    if tuple(v.shape) != (batch, n):
        raise ValueError("u and v must both be [batch][n]")
    if out is None:
        out = np.empty((batch, 2 * n), dtype=np.uint32)
    if tuple(out.shape) != (batch, 2 * n):
        raise ValueError(f"out must have shape {(batch, 2 * n)}")
    p = plan(B, t4, t3, chunk)
    st = lib().toom_mul_batched_host(ptr(out), ptr(u), ptr(v), n, batch, ctypes.byref(p), _stream(stream))
    _check(st, "toom_mul_batched_host")
    return out


def base_interleaved(u: torch.Tensor, v: torch.Tensor, stream=None) -> torch.Tensor:
    """Stage a3 alone: u, v interleaved [E][count] signed; returns [2E][count]."""
    E, count = u.shape
    out = torch.empty((2 * E, count), dtype=u.dtype, device=u.device)
    _check(lib().toom_base_interleaved(_dev(out, "out"), _dev(u, "u"), _dev(v, "v"), E, count, _stream(stream)),
           "toom_base_interleaved")
    return out


def base_interleaved_tc(u: torch.Tensor, v: torch.Tensor, stream=None) -> torch.Tensor:
    """Stage a3 on the int8 tensor cores (tcgen05 kind::i8):
    u, v interleaved [E][count] signed; returns [2E][count]."""
    E, count = u.shape
    out = torch.empty((2 * E, count), dtype=u.dtype, device=u.device)
    _check(lib().toom_base_interleaved_tc(_dev(out, "out"), _dev(u, "u"), _dev(v, "v"), E, count, _stream(stream)),
           "toom_base_interleaved_tc")
    return out


def eval_top(a: torch.Tensor, B: int, stream=None) -> torch.Tensor:
    """Stage a2 alone (top level): a [batch][n] unsigned -> [e][npoints*batch]
    interleaved two's complement values U(x_k) (column k*batch + i)."""
    batch, n = a.shape
    e = lib().toom_eval_width(n, B)
    npts = lib().toom_npoints(B)
    out = torch.empty((e, npts * batch), dtype=a.dtype, device=a.device)
    _check(lib().toom_eval_top(_dev(out, "out"), _dev(a, "a"), n, batch, B, _stream(stream)), "toom_eval_top")
    return out


def eval_points(a: torch.Tensor, B: int, signed: bool = False, stream=None) -> torch.Tensor:
    """Long-path stage a1+a2: a [batch][n] -> [2B-1][batch][e] values at the
    point set of B (two's complement)."""
    batch, n = a.shape
    e = lib().toom_eval_width(n, B)
    npts = lib().toom_npoints(B)
    out = torch.empty((npts, batch, e), dtype=a.dtype, device=a.device)
    _check(lib().toom_eval_points(_dev(out, "out"), _dev(a, "a"), n, batch, B, 1 if signed else 0, _stream(stream)),
           "toom_eval_points")
    return out


def eval_points_range(a: torch.Tensor, B: int, k0: int, k1: int, signed: bool = False, stream=None) -> torch.Tensor:
    """As eval_points for the points k0 <= k < k1: -> [k1-k0][batch][e]."""
    batch, n = a.shape
    e = lib().toom_eval_width(n, B)
    out = torch.empty((max(0, k1 - k0), batch, e), dtype=a.dtype, device=a.device)
    if k1 <= k0:
        return out
    _check(lib().toom_eval_points_range(_dev(out, "out"), _dev(a, "a"), n, batch, B, 1 if signed else 0, k0, k1,
                                        _stream(stream)),
           "toom_eval_points_range")
    return out


def interp_recompose(y: torch.Tensor, n: int, B: int, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Long-path stages a4+a5: y [2B-1][batch][2e] products -> w [batch][2n]."""
    npts, batch, w2 = y.shape
    if npts != lib().toom_npoints(B) or w2 != lib().toom_product_width_point(n, B):
        raise ValueError(f"y must be [{lib().toom_npoints(B)}][batch][{lib().toom_product_width_point(n, B)}]")
    if out is None:
        out = torch.empty((batch, 2 * n), dtype=y.dtype, device=y.device)
    _check(lib().toom_interp_recompose(_out(out, "out", (batch, 2 * n), y), _dev(y, "y"), n, batch, B,
                                       _stream(stream)),
           "toom_interp_recompose")
    return out


def mul_signed_batched(u: torch.Tensor, v: torch.Tensor, B: int = 4, t4: int = 256, t3: int = 64,
                       long_count: int = 0, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Two's-complement products w[i] = u[i]*v[i] ([batch][n] -> [batch][2n])."""
    if u.shape != v.shape or u.dim() != 2:
        raise ValueError("u and v must both be [batch][n]")
    batch, n = u.shape
    if out is None:
        out = torch.empty((batch, 2 * n), dtype=u.dtype, device=u.device)
    p = plan(B, t4, t3, 0, long_count)
    _check(lib().toom_mul_signed_batched(_out(out, "out", (batch, 2 * n), u), _dev(u, "u"), _dev(v, "v"), n, batch, ctypes.byref(p),
                                         _stream(stream)), "toom_mul_signed_batched")
    return out


def workspace_bytes(n: int, batch: int, B: int = 4, t4: int = 256, t3: int = 64, chunk: int = 0) -> int:
    p = plan(B, t4, t3, chunk)
    return lib().toom_workspace_bytes(n, batch, ctypes.byref(p))


def last_launch_count() -> int:
    return lib().toom_last_launch_count()


def plan_describe(n: int, batch: int, B: int = 4, t4: int = 256, t3: int = 64, chunk: int = 0,
                  long_count: int = 0) -> dict:
    import json
    p = plan(B, t4, t3, chunk, long_count)
    need = lib().toom_plan_describe(n, batch, ctypes.byref(p), None, 0)
    if not need:
        raise ValueError("invalid plan")
    buf = ctypes.create_string_buffer(need)
    lib().toom_plan_describe(n, batch, ctypes.byref(p), buf, need)
    return json.loads(buf.value.decode())


CATEGORIES = ("eval", "base", "interp", "other")


def set_fused(on: bool = True):
    """Use (default) or bypass the fused bottom-level kernel."""
    lib().toom_set_fused(1 if on else 0)


def set_top_stream(mode: int = 2):
    """Top-level interpolation kernel: 3 one warp per product (when the fused
    level is directly below), 2 smem-staged (default), 1 one-pass stream,
    0 per-row (all exact)."""
    lib().toom_set_top_stream(int(mode))


def profile_enable(on: bool = True):
    lib().toom_profile_enable(1 if on else 0)


def profile_collect() -> dict:
    ms = (ctypes.c_double * 4)()
    cnt = (ctypes.c_size_t * 4)()
    lib().toom_profile_collect(ms, cnt, 4)
    return {c: dict(ms=ms[i], launches=cnt[i]) for i, c in enumerate(CATEGORIES)}


def probe_limb_products(stream=None) -> tuple:
    """(limb-products/s, elapsed ms) of the integer-MAD peak probe
    (IMAD.WIDE.U32 issue rate)."""
    ms = ctypes.c_double(0)
    r = lib().toom_probe_limb_products(ctypes.byref(ms), _stream(stream))
    if r < 0:
        raise RuntimeError("probe failed")
    return r, ms.value


def probe_carry_chain(stream=None) -> tuple:
    """(limb-products/s, elapsed ms) of the mad.lo.cc/madc.hi.cc/addc sequence."""
    ms = ctypes.c_double(0)
    r = lib().toom_probe_carry_chain(ctypes.byref(ms), _stream(stream))
    if r < 0:
        raise RuntimeError("probe failed")
    return r, ms.value


def set_check(on: bool = True):
    """Device-side exact-division checks (a failure reads back as
    TOOM_EINEXACT from last_error())."""
    lib().toom_set_check(1 if on else 0)


def set_verify(on: bool = True):
    """Verify every unsigned result by its residue mod 2^61-1 on the device
    (a mismatch reads back as TOOM_EVERIFY from last_error())."""
    lib().toom_set_verify(1 if on else 0)


def debug_fault(kind: int = 0):
    """Fault injection for tests: 1 = flip one bit of one base-case product in
    the fused bottom kernel; 0 = off."""
    lib().toom_debug_fault(int(kind))


def last_error() -> int:
    """toom_last_error(): the sticky host status of this thread's last failed
    call, or a device-detected failure (TOOM_EINEXACT / TOOM_EVERIFY) when
    set_check / set_verify are on (synchronizes the device).  Clears it."""
    return lib().toom_last_error()


def set_t16_matrix(on: bool = True):
    """Toom-16 top-level interpolation: matrix form (default) or the staged
    Newton program."""
    lib().toom_set_t16_matrix(1 if on else 0)


def set_c2_mode(mode: int = 2):
    """C2-shaped batches: 2 = deferred bottom + one top division by 360^2
    (default), 1 = top division by 360 over per-row bottom, 0 = per-row both."""
    lib().toom_set_c2_mode(int(mode))


def set_lazy_bottom(on: bool = True):
    """Single large products: the Toom-3 bottom under the lazy levels hands up
    X = 6 y (default) or divides its rows itself."""
    lib().toom_set_lazy_bottom(1 if on else 0)


def toom_mul_ntt(u: torch.Tensor, v: torch.Tensor, B: int = 16, out: torch.Tensor | None = None,
                 stream=None) -> torch.Tensor:
    """Toom-B top level with its 2B-1 products by the NTT inner multiplier
    (B = 0: the NTT product alone); 1-D uint32 CUDA tensors, nu + nv limbs."""
    if u.dim() != 1 or v.dim() != 1 or u.dtype != v.dtype:
        raise ValueError("u and v must be 1-D tensors of one dtype")
    nu, nv = u.numel(), v.numel()
    if out is None:
        out = torch.empty(nu + nv, dtype=u.dtype, device=u.device)
    _check(lib().toom_mul_ntt(_out(out, "out", (nu + nv,), u), _dev(u, "u"), nu, _dev(v, "v"), nv, B,
                              _stream(stream)), "toom_mul_ntt")
    return out
