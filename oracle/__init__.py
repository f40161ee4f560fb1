"""oracle -- TEST INFRASTRUCTURE ONLY (see oracle/toom_oracle.c header).

Python loader for the plain-C oracle.  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference legs may import this package.
The product path (paper_1602_02740_b200/) never imports it.

Functions mirror toom_oracle.c:
  schoolbook(u, v)                 O1, the definition w = u*v
  toom(u, v, top_B, t4, t3)        O2, recursive Toom-Cook with the paper's
                                   points 0, +-2^j and the §3/§4 listings
  residue(a, p), is_prime(n),      O3, residues mod seeded 61-bit primes
  primes(seed, k)
  interp_listings(...), even_odd_interp(...)   the §3/§4 listings on values
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "toom_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# reference recursion shape (SURVEY.md §8 definitions): Toom-4 while n > 256,
# Toom-3 while n > 64, schoolbook at n <= 64.
T4_DEFAULT = 256
T3_DEFAULT = 64


def build(force: bool = False) -> str:
    """Compile toom_oracle.c with plain gcc -O2 (no intrinsics, no asm)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-Wall", "-shared", "-fPIC", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            P = ctypes.POINTER(ctypes.c_uint32)
            sz = ctypes.c_size_t
            L.oracle_schoolbook.argtypes = [P, sz, P, sz, P]
            L.oracle_schoolbook.restype = None
            L.oracle_schoolbook_batched.argtypes = [P, P, P, sz, sz]
            L.oracle_schoolbook_batched.restype = None
            L.oracle_toom.argtypes = [P, sz, P, sz, P, ctypes.c_int, sz, sz]
            L.oracle_toom.restype = ctypes.c_int
            L.oracle_toom_mt.argtypes = [P, sz, P, sz, P, ctypes.c_int, sz, sz, ctypes.c_int]
            L.oracle_toom_mt.restype = ctypes.c_int
            L.oracle_toom_batched.argtypes = [P, P, P, sz, sz, ctypes.c_int, sz, sz]
            L.oracle_toom_batched.restype = ctypes.c_int
            L.oracle_reset_counters.argtypes = []
            L.oracle_products_at_depth.argtypes = [ctypes.c_int]
            L.oracle_products_at_depth.restype = ctypes.c_long
            L.oracle_set_fault_skip_division.argtypes = [ctypes.c_int]
            L.oracle_interp_listings.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), P, sz, P, P]
            L.oracle_interp_listings.restype = ctypes.c_int
            L.oracle_even_odd_interp.argtypes = [ctypes.c_int, P, P, P, sz, P]
            L.oracle_even_odd_interp.restype = ctypes.c_int
            L.oracle_mod.argtypes = [P, sz, ctypes.c_uint64]
            L.oracle_mod.restype = ctypes.c_uint64
            L.oracle_is_prime_u64.argtypes = [ctypes.c_uint64]
            L.oracle_is_prime_u64.restype = ctypes.c_int
            L.oracle_alpha_exponent.argtypes = [ctypes.c_int]
            L.oracle_alpha_exponent.restype = ctypes.c_double
            _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _u32(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint32))


class InexactDivision(RuntimeError):
    """An 'exact' division left a remainder (SPEC.md:462 exit code 3)."""


def schoolbook(u, v) -> np.ndarray:
    u, v = _u32(u), _u32(v)
    w = np.zeros(u.size + v.size, dtype=np.uint32)
    lib().oracle_schoolbook(_p(u), u.size, _p(v), v.size, _p(w))
    return w


def schoolbook_batched(u, v) -> np.ndarray:
    u, v = _u32(u), _u32(v)
    batch, n = u.shape
    w = np.zeros((batch, 2 * n), dtype=np.uint32)
    lib().oracle_schoolbook_batched(_p(u), _p(v), _p(w), n, batch)
    return w


def toom(u, v, top_B: int = 0, t4: int = T4_DEFAULT, t3: int = T3_DEFAULT, threads: int = 1) -> np.ndarray:
    """O2 on one product; threads > 1 puts the 2B-1 top-level products on
    that many host threads (Eq. 2.5)."""
    u, v = _u32(u), _u32(v)
    w = np.zeros(u.size + v.size, dtype=np.uint32)
    if threads > 1:
        st = lib().oracle_toom_mt(_p(u), u.size, _p(v), v.size, _p(w), top_B, t4, t3, threads)
    else:
        st = lib().oracle_toom(_p(u), u.size, _p(v), v.size, _p(w), top_B, t4, t3)
    if st:
        raise InexactDivision(f"oracle_toom status {st}")
    return w


def toom_batched(u, v, top_B: int = 0, t4: int = T4_DEFAULT, t3: int = T3_DEFAULT,
                 threads: int = 1) -> np.ndarray:
    """Batched O2; products are split across `threads` host threads (ctypes
    releases the GIL), following Eq. 2.5's products-on-processors model."""
    u, v = _u32(u), _u32(v)
    batch, n = u.shape
    w = np.zeros((batch, 2 * n), dtype=np.uint32)
    L = lib()
    if threads <= 1 or batch <= 1:
        st = L.oracle_toom_batched(_p(u), _p(v), _p(w), n, batch, top_B, t4, t3)
        if st:
            raise InexactDivision(f"oracle_toom_batched status {st}")
        return w
    bounds = np.linspace(0, batch, threads + 1).astype(int)
    status = [0] * threads

    def run(t):
        a, b = bounds[t], bounds[t + 1]
        if b > a:
            status[t] = L.oracle_toom_batched(_p(u[a:b]), _p(v[a:b]), _p(w[a:b]), n, int(b - a), top_B, t4, t3)

    ths = [threading.Thread(target=run, args=(t,)) for t in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    if any(status):
        raise InexactDivision(f"oracle_toom_batched status {status}")
    return w


def reset_counters():
    lib().oracle_reset_counters()


def products_at_depth(d: int) -> int:
    return lib().oracle_products_at_depth(d)


def set_fault_skip_division(k: int):
    lib().oracle_set_fault_skip_division(k)


def _to_twos(vals, width):
    out = np.zeros((len(vals), width), dtype=np.uint32)
    mod = 1 << (32 * width)
    for i, x in enumerate(vals):
        x = int(x)
        assert -(mod >> 1) <= x < (mod >> 1)
        out[i] = np.frombuffer((x % mod).to_bytes(4 * width, "little"), dtype=np.uint32)
    return out


def _from_twos(arr, width):
    res = []
    mod = 1 << (32 * width)
    for row in arr:
        x = int.from_bytes(np.ascontiguousarray(row).tobytes(), "little")
        if x >= mod >> 1:
            x -= mod
        res.append(x)
    return res


def interp_listings(xs, ys, width: int = 16):
    """Run listing 1 then listing 2 on the points
    (xs[k], ys[k]); returns (alphas, coeffs) as Python ints."""
    n = len(xs) - 1
    x = np.asarray(xs, dtype=np.int64)
    y = _to_twos(ys, width)
    a = np.zeros_like(y)
    c = np.zeros_like(y)
    st = lib().oracle_interp_listings(n, x.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), _p(y), width, _p(a), _p(c))
    if st == 3:
        raise InexactDivision("listing division left a remainder")
    if st == 1:
        raise OverflowError("width too small")
    return _from_twos(a, width), _from_twos(c, width)


def even_odd_interp(y0, yplus, yminus, width: int = 16):
    """The §4 even-odd driver on W(0), W(2^j), W(-2^j); returns w_0..w_2n."""
    n = len(yplus)
    a0 = _to_twos([y0], width)
    ap = _to_twos(yplus, width) if n else np.zeros((0, width), np.uint32)
    am = _to_twos(yminus, width) if n else np.zeros((0, width), np.uint32)
    w = np.zeros((2 * n + 1, width), dtype=np.uint32)
    st = lib().oracle_even_odd_interp(n, _p(a0), _p(np.ascontiguousarray(ap)), _p(np.ascontiguousarray(am)), width, _p(w))
    if st == 3:
        raise InexactDivision("even-odd division left a remainder")
    if st == 1:
        raise OverflowError("width too small")
    return _from_twos(w, width)


def residue(a, p: int) -> int:
    a = _u32(a).ravel()
    return int(lib().oracle_mod(_p(a), a.size, p))


def is_prime(n: int) -> bool:
    return bool(lib().oracle_is_prime_u64(n))


def primes(seed: int, k: int = 8, bits: int = 61):
    """k distinct random `bits`-bit primes drawn from a seeded SplitMix64 stream
    (prime-selection seed 1602027499)."""
    from synth import sm64
    out, ctr = [], 0
    while len(out) < k:
        x = sm64((seed + ctr) & ((1 << 64) - 1))
        ctr += 1
        cand = (x >> (64 - bits)) | (1 << (bits - 1)) | 1
        if is_prime(cand) and cand not in out:
            out.append(cand)
    return out


def alpha_exponent(B: int) -> float:
    return lib().oracle_alpha_exponent(B)
