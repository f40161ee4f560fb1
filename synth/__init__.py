"""Seeded synthetic inputs for every config -- shared by the oracle side and the
CUDA side.  This module holds NONE of the method's arithmetic: it only draws
limbs from a counter-based generator and lays out the configs' input classes.

Generator (SURVEY.md §8(d) "PRNG"): SplitMix64's finalizer, keyed by
(seed, product i, operand o, limb pair j//2).  Limb j is the low 32 bits of
word j//2 for even j and the high 32 bits for odd j.

    sm64(x)    = finalizer(x + 0x9E3779B97F4A7C15)
    key(i, o)  = sm64(sm64(seed) ^ (2*i + o))
    word(i,o,p)= sm64(key(i, o) ^ (p * 0xD6E8FEB86659FD93))

Seeds: seed_Ck = 1602027400 + k (k = 1..5), BASELINE.md §2.

Config input classes:
  C1: 256 uniform pairs of 96 limbs + 4 edge pairs u = v = e,
      e in {2^3072-1, 0, 1, 2^3071} (batch indices 256..259)
  C2: 65536 uniform pairs of 256 limbs
  C3: 4096 pairs of 2048 limbs in contiguous quarters: all-0xFFFFFFFF (u=v),
      alternating 0/0xFFFFFFFF (limb i = 0 for even i; u=v), single random
      bit (u = 2^a, v = 2^c), uniform
  C4: one uniform pair of 2^20 limbs
  C5: one uniform pair of 2^24 limbs
"""
from __future__ import annotations

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15
C_MUL1 = 0xBF58476D1CE4E5B9
C_MUL2 = 0x94D049BB133111EB
C_PAIR = 0xD6E8FEB86659FD93

SEED_BASE = 1602027400
PRIME_SEED = 1602027499


def seed_for(config: int) -> int:
    return SEED_BASE + config


def _sm64_np(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(C_MUL1)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(C_MUL2)
        return z ^ (z >> np.uint64(31))


def sm64(x: int) -> int:
    z = (x + GOLDEN) & M64
    z = ((z ^ (z >> 30)) * C_MUL1) & M64
    z = ((z ^ (z >> 27)) * C_MUL2) & M64
    return z ^ (z >> 31)


def uniform_limbs(seed: int, first_product: int, count: int, operand: int, n: int) -> np.ndarray:
    """uint32 array [count][n]: limbs of operand `operand` of products
    first_product .. first_product+count-1."""
    if count == 0 or n == 0:
        return np.zeros((count, n), dtype=np.uint32)
    s = np.uint64(sm64(seed & M64))
    i = np.arange(first_product, first_product + count, dtype=np.uint64)
    key = _sm64_np(s ^ (np.uint64(2) * i + np.uint64(operand)))          # [count]
    npairs = (n + 1) // 2
    p = np.arange(npairs, dtype=np.uint64)
    with np.errstate(over="ignore"):
        pk = p * np.uint64(C_PAIR)
    words = _sm64_np(key[:, None] ^ pk[None, :])                         # [count][npairs]
    limbs = words.view(np.uint32).reshape(count, 2 * npairs)             # little-endian: lo, hi
    return np.ascontiguousarray(limbs[:, :n])


def uniform_limbs_chunked(seed: int, count: int, operand: int, n: int, chunk: int = 4096) -> np.ndarray:
    out = np.empty((count, n), dtype=np.uint32)
    for a in range(0, count, chunk):
        b = min(count, a + chunk)
        out[a:b] = uniform_limbs(seed, a, b - a, operand, n)
    return out


def _long_uniform(seed: int, operand: int, n: int, chunk: int = 1 << 22) -> np.ndarray:
    """One long operand (C4/C5): product index 0, limb pairs generated in chunks."""
    s = np.uint64(sm64(seed & M64))
    key = _sm64_np(np.array([s ^ np.uint64(operand)], dtype=np.uint64))[0]
    npairs = (n + 1) // 2
    out = np.empty(2 * npairs, dtype=np.uint32)
    for a in range(0, npairs, chunk):
        b = min(npairs, a + chunk)
        p = np.arange(a, b, dtype=np.uint64)
        with np.errstate(over="ignore"):
            w = _sm64_np(key ^ (p * np.uint64(C_PAIR)))
        out[2 * a:2 * b] = w.view(np.uint32)
    return out[:n]


def config_inputs(config: int, batch: int | None = None, first: int = 0):
    """(u, v) uint32 arrays for config C1..C5.

    For the batched configs (1..3) returns [batch][n] arrays; `batch`/`first`
    select a sub-range of the config's batch (products first..first+batch-1)
    so shards and bounded samples see exactly the same values as the full run.
    For C4/C5 returns 1-D arrays of n limbs.
    """
    seed = seed_for(config)
    if config == 1:
        n, total = 96, 260
        batch = total - first if batch is None else batch
        u = np.zeros((batch, n), dtype=np.uint32)
        v = np.zeros((batch, n), dtype=np.uint32)
        for r in range(batch):
            i = first + r
            if i < 256:
                u[r] = uniform_limbs(seed, i, 1, 0, n)[0]
                v[r] = uniform_limbs(seed, i, 1, 1, n)[0]
            else:
                e = c1_edge(i - 256, n)
                u[r] = e
                v[r] = e
        return u, v
    if config == 2:
        n, total = 256, 65536
        batch = total - first if batch is None else batch
        u = np.empty((batch, n), dtype=np.uint32)
        v = np.empty((batch, n), dtype=np.uint32)
        for a in range(0, batch, 4096):
            b = min(batch, a + 4096)
            u[a:b] = uniform_limbs(seed, first + a, b - a, 0, n)
            v[a:b] = uniform_limbs(seed, first + a, b - a, 1, n)
        return u, v
    if config == 3:
        n, total = 2048, 4096
        batch = total - first if batch is None else batch
        u = np.empty((batch, n), dtype=np.uint32)
        v = np.empty((batch, n), dtype=np.uint32)
        for r in range(batch):
            i = first + r
            cls = c3_class(i, total)
            if cls == 0:
                u[r] = 0xFFFFFFFF
                v[r] = 0xFFFFFFFF
            elif cls == 1:
                pat = np.zeros(n, dtype=np.uint32)
                pat[1::2] = 0xFFFFFFFF
                u[r] = pat
                v[r] = pat
            elif cls == 2:
                a, c = c3_bits(seed, i, n)
                u[r] = 0
                v[r] = 0
                u[r, a // 32] = np.uint32(1 << (a % 32))
                v[r, c // 32] = np.uint32(1 << (c % 32))
            else:
                u[r] = uniform_limbs(seed, i, 1, 0, n)[0]
                v[r] = uniform_limbs(seed, i, 1, 1, n)[0]
        return u, v
    if config == 4:
        n = 1 << 20
        return _long_uniform(seed, 0, n), _long_uniform(seed, 1, n)
    if config == 5:
        n = 1 << 24
        return _long_uniform(seed, 0, n), _long_uniform(seed, 1, n)
    raise ValueError(f"unknown config C{config}")


def c1_edge(k: int, n: int = 96) -> np.ndarray:
    """C1 edge values: 2^3072-1, 0, 1, 2^3071."""
    e = np.zeros(n, dtype=np.uint32)
    if k == 0:
        e[:] = 0xFFFFFFFF
    elif k == 1:
        pass
    elif k == 2:
        e[0] = 1
    elif k == 3:
        e[n - 1] = 0x80000000
    else:
        raise ValueError(k)
    return e


def c3_class(i: int, total: int = 4096) -> int:
    """0 all-ones, 1 alternating, 2 single-bit, 3 uniform (contiguous quarters)."""
    return min(3, (4 * i) // total)


def c3_bits(seed: int, i: int, n: int = 2048):
    """bit positions a, c of the single-bit class, uniform in [0, 32n)."""
    w = sm64(sm64(seed) ^ (0x5B17 << 32) ^ i)
    nbits = 32 * n
    return int(w & 0xFFFFFFFF) % nbits, int(w >> 32) % nbits


CONFIGS = {
    1: dict(name="C1", n=96, batch=260, B=3),
    2: dict(name="C2", n=256, batch=65536, B=4),
    3: dict(name="C3", n=2048, batch=4096, B=8),
    4: dict(name="C4", n=1 << 20, batch=1, B=4),
    5: dict(name="C5", n=1 << 24, batch=1, B=16),
}


def to_int(limbs) -> int:
    """Python int from a little-endian uint32 limb array (for tests)."""
    a = np.ascontiguousarray(np.asarray(limbs, dtype=np.uint32))
    return int.from_bytes(a.tobytes(), "little")


def from_int(x: int, n: int) -> np.ndarray:
    """little-endian uint32 limbs of a non-negative int (for tests)."""
    return np.frombuffer(x.to_bytes(4 * n, "little"), dtype=np.uint32).copy()
