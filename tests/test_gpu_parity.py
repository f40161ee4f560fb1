"""GPU parity tests: the CUDA path (through the C ABI) against the CPU oracle,
element by element on the same seeded inputs.  Integer work: the bar is
bit-exact.  Run on a B200 with  python -m pytest tests -m gpu.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

tg = pytest.importorskip("paper_1602_02740_b200")
I = synth.to_int


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")
    tg.lib()


PRIMES = None


def primes():
    global PRIMES
    if PRIMES is None:
        PRIMES = oracle.primes(synth.PRIME_SEED, 8)
    return PRIMES


def check_residues(u, v, w):
    for p in primes():
        assert oracle.residue(w, p) == oracle.residue(u, p) * oracle.residue(v, p) % p


# ------------------------------------------------------------ stage a3 alone


@pytest.mark.parametrize("E", [1, 2, 5, 17, 18, 23, 33, 40, 41, 64])
def test_base_case_signed_interleaved(E):
    rng = np.random.default_rng(E)
    count = 1000 + E
    a = rng.integers(0, 2**32, (E, count), dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, (E, count), dtype=np.uint64).astype(np.uint32)
    a[:, 0] = 0xFFFFFFFF            # -1
    b[:, 1] = 0                     # 0
    a[:, 2] = 0
    a[E - 1, 2] = 0x80000000        # most negative
    b[:, 2] = a[:, 2]
    w = host(tg.base_interleaved(dev(a), dev(b)))

    def sval(col):
        x = I(col)
        return x - (1 << (32 * len(col))) if x >> (32 * len(col) - 1) else x

    for c in list(range(8)) + list(rng.integers(0, count, 64)):
        x, y = sval(a[:, c]), sval(b[:, c])
        # oracle: schoolbook on the magnitudes, sign applied
        mag = I(oracle.schoolbook(synth.from_int(abs(x), E), synth.from_int(abs(y), E)))
        want = mag if (x < 0) == (y < 0) else -mag
        assert sval(w[:, c]) == want


@pytest.mark.parametrize("E", [2, 5, 9, 16, 17, 18, 23, 24])
def test_base_case_tensor_core_int8(E):
    """the base case on tcgen05 kind::i8 (Toeplitz byte windows
    x reversed 32-byte chunks, s32 accumulation in TMEM) equals the IMAD.WIDE
    path element by element, and the oracle's schoolbook (w = uv
    is unique) on sampled products, adversarial magnitudes included (all-ones
    bytes give the largest partial sums, 32 * 255^2 per MMA output)."""
    rng = np.random.default_rng(100 + E)
    count = 3000 + E
    a = rng.integers(0, 2**32, (E, count), dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, (E, count), dtype=np.uint64).astype(np.uint32)
    a[:, 0] = 0xFFFFFFFF            # -1
    b[:, 1] = 0                     # 0
    a[:, 2] = 0
    a[E - 1, 2] = 0x80000000        # most negative
    b[:, 2] = a[:, 2]
    a[:, 3] = 0xFFFFFFFF            # |x| = 2^(32E-1) - 1: all-ones magnitude bytes
    a[E - 1, 3] = 0x7FFFFFFF
    b[:, 3] = a[:, 3]
    got = host(tg.base_interleaved_tc(dev(a), dev(b)))
    assert np.array_equal(got, host(tg.base_interleaved(dev(a), dev(b))))

    def sval(col):
        x = I(col)
        return x - (1 << (32 * len(col))) if x >> (32 * len(col) - 1) else x

    for c in list(range(8)) + list(rng.integers(0, count, 32)):
        x, y = sval(a[:, c]), sval(b[:, c])
        mag = I(oracle.schoolbook(synth.from_int(abs(x), E), synth.from_int(abs(y), E)))
        want = mag if (x < 0) == (y < 0) else -mag
        assert sval(got[:, c]) == want


def test_base_case_tensor_core_rejects_unsupported_width():
    a = torch.zeros((40, 4), dtype=torch.uint32, device="cuda")
    with pytest.raises(RuntimeError):
        tg.base_interleaved_tc(a, a)


# ------------------------------------------------------------ stage a2 alone


@pytest.mark.parametrize("B,n", [(3, 96), (4, 256), (4, 250), (8, 2048), (3, 7), (8, 100)])
def test_eval_top_matches_definition(B, n):
    pts = {3: [(0, 1), (1, 1), (-1, 1), (2, 1), (1, 0)],
           4: [(0, 1), (1, 1), (-1, 1), (2, 1), (-2, 1), (1, 2), (1, 0)],
           8: [(0, 1)] + [(s * (1 << j), 1) for j in range(7) for s in (1, -1)]}[B]
    batch = 37
    u, _ = synth.config_inputs(2, batch=batch)
    u = np.ascontiguousarray(np.resize(u, (batch, n)))
    u[0] = 0xFFFFFFFF
    out = host(tg.eval_top(dev(u), B))
    e = out.shape[0]
    b = -(-n // B)
    for i in (0, 1, batch - 1):
        blocks = [I(u[i, k * b:min(n, (k + 1) * b)]) for k in range(B)]
        for k, (p, q) in enumerate(pts):
            want = sum(x * p**j * q ** (B - 1 - j) for j, x in enumerate(blocks))
            col = out[:, k * batch + i]
            got = I(col)
            if got >> (32 * e - 1):
                got -= 1 << (32 * e)
            assert got == want


# ------------------------------------------------------------ configs


def run_batched(u, v, B, t4=256, t3=64, chunk=0, long_count=0):
    w = tg.toom_mul_batched(dev(u), dev(v), B=B, t4=t4, t3=t3, chunk=chunk, long_count=long_count)
    torch.cuda.synchronize()
    return host(w)


def test_c1_full_bit_exact():
    u, v = synth.config_inputs(1)
    w = run_batched(u, v, 3, t4=10**9, t3=10**9)       # one Toom-3 level, schoolbook base
    want = oracle.toom_batched(u, v, top_B=3, t4=10**9, t3=64, threads=8)
    assert np.array_equal(w, want)
    # edge pairs (SURVEY §8(c) reading 16): closed forms
    for k, expect in enumerate([(2**3072 - 1) ** 2, 0, 1, 2**6142]):
        assert I(w[256 + k]) == expect


C2_PLAN = dict(t4=32, t3=32)   # "Toom-4 ... recursing to a 32-limb schoolbook base"


def test_c2_slice_bit_exact():
    u, v = synth.config_inputs(2, batch=3000, first=1000)
    w = run_batched(u, v, 4, **C2_PLAN)
    want = oracle.toom_batched(u, v, top_B=4, threads=8)
    assert np.array_equal(w, want)


def test_c2_full_batch_bit_exact():
    """The bench launch configuration: all 65536 products of BASELINE configs[1]
    in one call, every product compared with the oracle O2 (w = uv
    is unique), plus residues on a sample."""
    import os
    u, v = synth.config_inputs(2)
    w = run_batched(u, v, 4, **C2_PLAN)
    want = oracle.toom_batched(u, v, top_B=4, threads=os.cpu_count() or 8)
    bad = np.nonzero((w != want).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} of 65536 products differ, first {bad[:8]}"
    rng = np.random.default_rng(2)
    for i in rng.integers(0, 65536, 16):
        check_residues(u[i], v[i], w[i])


@pytest.mark.parametrize("batch", [1, 29, 1234])
def test_c2_modes_equal_oracle(batch):
    """The three C2 paths (reading 18): 2 = bottom with the deferred
    common denominator + top level as one division by 360^2 (csrc/fused_c2.cuh,
    csrc/toplevel_cls.cuh), 1 = per-row bottom + one top division by 360,
    0 = per-row divisions at both levels; all equal to the oracle, with
    extreme operands (all-ones: the largest evaluated values and products,
    carries through whole segments; alternating limbs; zero; one top bit) and
    ragged CTA tails (28 products per top CTA, 32 children per bottom CTA)."""
    rng = np.random.default_rng(batch)
    n = 256
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    pats = [np.full(n, 0xFFFFFFFF, np.uint32), np.tile(np.array([0, 0xFFFFFFFF], np.uint32), n // 2),
            np.zeros(n, np.uint32), np.r_[np.zeros(n - 1, np.uint32), np.uint32(1 << 31)]]
    for i in range(min(batch, 16)):
        u[i] = pats[i % 4]
        v[i] = pats[(i // 4) % 4]
    want = oracle.schoolbook_batched(u, v)
    try:
        for mode in (2, 1, 0):
            tg.set_c2_mode(mode)
            w = run_batched(u, v, 4, **C2_PLAN)
            bad = np.nonzero((w != want).any(axis=1))[0]
            assert bad.size == 0, f"mode {mode}: {bad.size} products differ, first {bad[:8]}"
    finally:
        tg.set_c2_mode(2)


@pytest.mark.parametrize("n", [1 << 16, 65538, 1 << 18])
def test_lazy_bottom_deferred_equals_per_row_and_oracle(n):
    """Single large products (the C4 recursion: lazy Toom-4 levels over the
    Toom-3 bottom of 66-limb parents): the bottom handing X = 6 y into the
    lazy block's finishing division (csrc/fused_dc.cuh, DESIGN.md readings
    18-19) against the per-row bottom and the oracle, uniform and adversarial
    operands."""
    rng = np.random.default_rng(n)
    a = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    b[: n // 3] = 0xFFFFFFFF
    a[n // 2: n // 2 + 999] = 0
    assert tg.plan_describe(n, 1, B=4)["lazy_bottom_dc"]
    want = oracle.toom(a, b, top_B=4)
    try:
        for on in (True, False):
            tg.set_lazy_bottom(on)
            w = host(tg.toom_mul(dev(a), dev(b), B=4))
            assert np.array_equal(w, want), on
            check_residues(a, b, w)
    finally:
        tg.set_lazy_bottom(True)


def test_c2_chunked_equals_unchunked():
    u, v = synth.config_inputs(2, batch=5000)
    a = run_batched(u, v, 4, **C2_PLAN)
    b = run_batched(u, v, 4, chunk=1024, **C2_PLAN)
    assert np.array_equal(a, b)


def test_c3_every_product_closed_forms_and_oracle():
    """BASELINE configs[2] in full (4096 products, one call): every product of
    the three structured quarters against its closed form,
    every uniform product against the oracle O2."""
    import os
    u, v = synth.config_inputs(3)
    w = run_batched(u, v, 8)
    n, N = 2048, 65536
    # all-ones quarter: (2^N - 1)^2 = 2^2N - 2^(N+1) + 1
    ones = synth.from_int((1 << (2 * N)) - (1 << (N + 1)) + 1, 2 * n)
    assert (w[0:1024] == ones[None, :]).all()
    # alternating quarter: u = v, (2^32 + 1)^2 w = 2^64 (2^N - 1)^2
    alt_u = I(u[1024])
    alt = synth.from_int(alt_u * alt_u, 2 * n)
    assert (2**32 + 1) ** 2 * I(alt) == 2**64 * (2**N - 1) ** 2
    assert (u[1024:2048] == u[1024][None, :]).all() and (v[1024:2048] == u[1024][None, :]).all()
    assert (w[1024:2048] == alt[None, :]).all()
    # single-bit quarter: 2^(a+c), one nonzero limb
    for i in range(2048, 3072):
        a, c = synth.c3_bits(synth.seed_for(3), i)
        e = a + c
        row = w[i]
        nz = np.flatnonzero(row)
        assert nz.tolist() == [e // 32] and int(row[e // 32]) == 1 << (e % 32), i
    # uniform quarter: the oracle on every product
    want = oracle.toom_batched(u[3072:], v[3072:], top_B=8, threads=os.cpu_count() or 8)
    bad = np.nonzero((w[3072:] != want).any(axis=1))[0]
    assert bad.size == 0, f"{bad.size} uniform products differ"
    for i in range(0, 4096, 257):
        check_residues(u[i], v[i], w[i])


def test_c3_small_slice_bit_exact_all_classes():
    idx = [0, 1, 1024, 1025, 2048, 2049, 4094, 4095]
    u, v = synth.config_inputs(3)
    u, v = u[idx], v[idx]
    w = run_batched(u, v, 8)
    assert np.array_equal(w, oracle.toom_batched(u, v, top_B=8, threads=8))


# ------------------------------------------------------------ edge cases


@pytest.mark.parametrize("B", [3, 4, 8])
@pytest.mark.parametrize("n", [16, 17, 31, 65, 100, 129, 257, 300])
def test_ragged_sizes(B, n):
    if n < 2 * B:
        pytest.skip("below the smallest Toom split")
    rng = np.random.default_rng(n * 10 + B)
    batch = 33
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    v[0] = 0xFFFFFFFF
    u[1] = 0
    for t4, t3 in [(256, 64), (8, 8)]:
        w = run_batched(u, v, B, t4=t4, t3=t3)
        assert np.array_equal(w, oracle.schoolbook_batched(u, v)), (B, n, t4, t3)


def test_empty_batch_and_errors():
    u = torch.zeros((0, 96), dtype=torch.uint32, device="cuda")
    w = tg.toom_mul_batched(u, u, B=3)
    assert w.shape == (0, 192)
    x = torch.zeros((4, 96), dtype=torch.uint32, device="cuda")
    with pytest.raises(tg.ToomError) as ei:
        tg.toom_mul_batched(x, x, B=5)
    assert ei.value.status == tg.TOOM_EINVAL
    big = torch.zeros(4 * 192 + 96, dtype=torch.uint32, device="cuda")
    with pytest.raises(tg.ToomError) as ei:                  # aliasing: w overlaps u
        tg.toom_mul_batched(big[96:96 + 384].view(4, 96), x, B=3, out=big[:768].view(4, 192))
    assert ei.value.status == tg.TOOM_EINVAL
    with pytest.raises(ValueError):                         # wrong output shape
        tg.toom_mul_batched(x, x, B=3, out=x.view(2, 192))
    with pytest.raises(TypeError):
        tg.toom_mul_batched(x.cpu(), x.cpu(), B=3)            # no CPU fallback


def test_toom_mul_unbalanced_and_zero_length():
    rng = np.random.default_rng(9)
    for nu, nv in [(300, 120), (97, 1000), (1, 64), (500, 500)]:
        a = rng.integers(0, 2**32, nu, dtype=np.uint64).astype(np.uint32)
        b = rng.integers(0, 2**32, nv, dtype=np.uint64).astype(np.uint32)
        for B in (3, 4, 8):
            w = host(tg.toom_mul(dev(a), dev(b), B=B))
            assert np.array_equal(w, oracle.schoolbook(a, b))
    z = torch.zeros(0, dtype=torch.uint32, device="cuda")
    a = dev(np.arange(5, dtype=np.uint32))
    assert not host(tg.toom_mul(a, z, B=4)).any()


def test_c4_single_large_product():
    u, v = synth.config_inputs(4)
    w = host(tg.toom_mul(dev(u), dev(v), B=4))
    check_residues(u, v, w)
    assert np.array_equal(w, oracle.toom(u, v, threads=8))


# ------------------------------------------------------------ fused bottom level


FUSED_SHAPES = [  # (B, n, t4, t3): bottom Toom levels with base widths 6, 9, 18, 23, 27, 33
    (3, 13, 256, 64), (4, 19, 256, 64), (3, 23, 256, 64), (4, 31, 256, 64), (3, 50, 256, 64),
    (4, 66, 256, 64), (3, 65, 256, 64), (4, 88, 256, 64), (3, 78, 256, 64), (3, 96, 10**9, 10**9),
    (4, 256, 32, 32), (4, 1024, 256, 64), (8, 2048, 256, 64), (4, 1040, 256, 64), (3, 500, 256, 20),
]


@pytest.mark.parametrize("B,n,t4,t3", FUSED_SHAPES)
def test_fused_bottom_equals_staged_and_oracle(B, n, t4, t3):
    rng = np.random.default_rng(n * 7 + B)
    batch = 70
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    v[0] = 0xFFFFFFFF
    u[1] = 0
    u[2, ::2] = 0
    v[2] = u[2]
    info = tg.plan_describe(n, batch, B=B, t4=t4, t3=t3)
    try:
        tg.set_fused(False)
        staged = run_batched(u, v, B, t4=t4, t3=t3)
    finally:
        tg.set_fused(True)
    fused = run_batched(u, v, B, t4=t4, t3=t3)
    want = oracle.schoolbook_batched(u, v)
    assert np.array_equal(staged, want), ("staged", info)
    assert np.array_equal(fused, want), ("fused", info)


def test_c2_plan_uses_fused_bottom():
    info = tg.plan_describe(256, 65536, B=4, t4=32, t3=32)
    assert info["fused_bottom"] and info["levels"][-1]["n"] == 18


# ------------------------------------------------------------ long-vector levels (C4/C5 upper levels)


@pytest.mark.parametrize("B", [3, 4, 8, 16])
@pytest.mark.parametrize("n", [40, 257, 1500, 5000, 20011])
def test_long_path_single_product(B, n):
    """toom_mul on one product: the upper levels run on the limb-parallel
    long-vector kernels (several tiles per vector at n >= 2048, ragged tail)."""
    if n < 2 * B:
        pytest.skip("below the smallest split")
    rng = np.random.default_rng(n + B)
    a = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    info = tg.plan_describe(n, 1, B=B)
    assert info["levels"][0]["long"] or info["levels"][0]["B"] != B or n <= 2048
    w = host(tg.toom_mul(dev(a), dev(b), B=B))
    assert np.array_equal(w, oracle.schoolbook(a, b)), info
    # the same product with every Toom level forced onto the long path
    w2 = host(tg.toom_mul_batched(dev(a[None]), dev(b[None]), B=B, long_count=1 << 30))
    assert np.array_equal(w2[0], w), info


@pytest.mark.parametrize("B", [3, 4, 8, 16])
def test_long_path_adversarial_carries(B):
    """all-ones, alternating, single-bit and zero-top operands: long carry and
    borrow chains across tiles (every limb 0xFFFFFFFF propagates)."""
    n = 9000
    ones = np.full(n, 0xFFFFFFFF, np.uint32)
    alt = np.zeros(n, np.uint32)
    alt[1::2] = 0xFFFFFFFF
    bit = np.zeros(n, np.uint32)
    bit[n // 3] = 1 << 7
    low = np.zeros(n, np.uint32)
    low[: n // 2] = 0xFFFFFFFF
    cases = [(ones, ones), (alt, alt), (bit, ones), (low, ones), (ones, low)]
    for a, b in cases:
        w = host(tg.toom_mul(dev(a), dev(b), B=B))
        assert I(w) == I(a) * I(b)


@pytest.mark.parametrize("B,n", [(3, 300), (4, 1000), (8, 2048), (4, 4100)])
def test_long_vs_short_levels_batched(B, n):
    """The same batch with the upper levels forced long (long_count large) and
    forced instance-parallel (long_count=1): identical to the oracle."""
    rng = np.random.default_rng(n * 3 + B)
    batch = 9
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    v[0] = 0xFFFFFFFF
    want = oracle.schoolbook_batched(u, v)
    for lc in (1, 1 << 30):
        w = host(tg.toom_mul_batched(dev(u), dev(v), B=B, long_count=lc))
        assert np.array_equal(w, want), lc


def test_c5_shape_reduced():
    """C5's top level (31-point Toom-16, homogeneous points) at 2^16 limbs,
    recursing with Toom-4/3: bit-exact against the oracle's own recursive Toom
    (paper points) and residues."""
    seed = synth.seed_for(5)
    n = 1 << 16
    u = synth.uniform_limbs(seed, 7, 1, 0, n)[0]
    v = synth.uniform_limbs(seed, 7, 1, 1, n)[0]
    w = host(tg.toom_mul(dev(u), dev(v), B=16))
    check_residues(u, v, w)
    assert np.array_equal(w, oracle.toom(u, v, top_B=16))


def test_c5_full():
    """configs[4] at full size: residues mod 8 seeded 61-bit primes (the
    oracle's recursive Toom at 2^24 limbs is test_c5_full_oracle, slow)."""
    u, v = synth.config_inputs(5)
    w = host(tg.toom_mul(dev(u), dev(v), B=16))
    check_residues(u, v, w)
    # closed-form spot check on the low and high limbs: w mod 2^64 and the top word
    assert I(w[:2]) == (I(u[:2]) * I(v[:2])) % (1 << 64)


def test_c5_full_oracle():
    """configs[4] at full size, bit-exact against the oracle's recursive Toom
    (the paper's points 0, +-2^j at the top; about 50 s on the
    box's host cores)."""
    import os
    u, v = synth.config_inputs(5)
    w = host(tg.toom_mul(dev(u), dev(v), B=16))
    assert np.array_equal(w, oracle.toom(u, v, top_B=16, threads=os.cpu_count() or 8))


# ------------------------------------------------------------ long-path stage exports + sharded C5


@pytest.mark.parametrize("B,n", [(16, 5000), (4, 3001), (3, 2500), (8, 4100)])
def test_stage_exports_compose(B, n):
    """eval_points -> per-point signed products -> interp_recompose == u*v,
    with the evaluation (eval_points_range, equal to the slices of
    eval_points) and the products in rank-sized shards (single-GPU emulation
    of the P=8 partition of dist.sharded_mul; ranks do not wait on one
    another)."""
    from paper_1602_02740_b200 import dist as tgdist
    rng = np.random.default_rng(B * 1000 + n)
    u = rng.integers(0, 2**32, (1, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (1, n), dtype=np.uint64).astype(np.uint32)
    U = tg.eval_points(dev(u), B)
    V = tg.eval_points(dev(v), B)
    npts = U.shape[0]
    Ys = []
    bounds, _ = tgdist.shard_bounds(npts, 8)
    for lo, hi in bounds:
        # each rank evaluates its own points (toom_eval_points_range) ...
        Ur = tg.eval_points_range(dev(u), B, lo, hi)
        Vr = tg.eval_points_range(dev(v), B, lo, hi)
        assert torch.equal(Ur, U[lo:hi]) and torch.equal(Vr, V[lo:hi])
        if hi > lo:   # ... and multiplies them
            Ys.append(tg.mul_signed_batched(Ur[:, 0].contiguous(), Vr[:, 0].contiguous(), B=4))
    Y = torch.cat([y.view(torch.int32) for y in Ys]).view(torch.uint32)
    w = host(tg.interp_recompose(Y.view(npts, 1, -1).contiguous(), n, B))
    assert np.array_equal(w[0], oracle.schoolbook(u[0], v[0]))


def test_signed_batched_products():
    rng = np.random.default_rng(77)
    n, batch = 3000, 5
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[1, -1] |= 0x80000000          # negative
    v[2] = 0xFFFFFFFF               # -1
    w = host(tg.mul_signed_batched(dev(u), dev(v), B=4))

    def sv(a):
        x = I(a)
        return x - (1 << (32 * len(a))) if int(a[-1]) >> 31 else x

    for i in range(batch):
        assert sv(w[i]) == sv(u[i]) * sv(v[i])


def test_sharded_mul_single_rank_cuda():
    from paper_1602_02740_b200 import dist as tgdist
    seed = synth.seed_for(5)
    n = 1 << 15
    u = synth.uniform_limbs(seed, 11, 1, 0, n)[0]
    v = synth.uniform_limbs(seed, 11, 1, 1, n)[0]
    w = host(tgdist.sharded_mul(dev(u), dev(v), n, tgdist.CudaOps()))
    assert np.array_equal(w, host(tg.toom_mul(dev(u), dev(v), B=16)))
    check_residues(u, v, w)


@pytest.mark.parametrize("B,n,t4,t3", [(3, 96, 10**9, 10**9), (4, 256, 32, 32), (4, 250, 32, 32), (3, 301, 256, 64),
                                       (4, 1000, 256, 64), (3, 13, 256, 64), (3, 96, 24, 24), (4, 120, 24, 24),
                                       (4, 520, 130, 130)])
def test_top_stream_vs_rows(B, n, t4, t3):
    rng = np.random.default_rng(n + 17 * B)
    batch = 77
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    v[0] = 0xFFFFFFFF
    u[1] = 0
    want = oracle.schoolbook_batched(u, v)
    try:
        for mode in (0, 1, 2, 3, 4):
            tg.set_top_stream(mode)
            got = run_batched(u, v, B, t4=t4, t3=t3, long_count=1)
            assert np.array_equal(got, want), mode
    finally:
        tg.set_top_stream(2)


@pytest.mark.parametrize("n", [2048, 1500, 777])
def test_p8_top_rows_vs_half_programs(n):
    """C3's top level (the paper's Toom-8 points): the row-parallel
    interpolation + segment recomposition against the one-lane-per-half
    streaming kernel and the oracle."""
    rng = np.random.default_rng(n)
    batch = 40
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    v[0] = 0xFFFFFFFF
    u[1, 1::2] = 0xFFFFFFFF
    u[1, ::2] = 0
    v[1] = u[1]
    want = oracle.schoolbook_batched(u, v)
    try:
        for mode in (0, 2):
            tg.set_top_stream(mode)
            got = run_batched(u, v, 8, long_count=1)
            assert np.array_equal(got, want), mode
    finally:
        tg.set_top_stream(2)


@pytest.mark.parametrize("B,n,t4,t3", [(4, 1026, 256, 64), (3, 300, 64, 64), (4, 4100, 256, 64), (3, 66, 10, 10)])
def test_rows_interp_lower_levels(B, n, t4, t3):
    """Signed lower levels: the row-parallel interpolation + segment
    recomposition (sign fills of negative coefficients) against the
    per-thread streaming programs (mode 0) and the oracle."""
    rng = np.random.default_rng(n * 5 + B)
    batch = 50
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    v[0] = 0xFFFFFFFF
    u[1, ::2] = 0
    u[2] = 0
    u[2, -1] = 1
    want = oracle.schoolbook_batched(u, v)
    try:
        for mode in (0, 2, 4):
            tg.set_top_stream(mode)   # 4: row-parallel lower levels
            got = run_batched(u, v, B, t4=t4, t3=t3, long_count=1)
            assert np.array_equal(got, want), mode
    finally:
        tg.set_top_stream(2)


@pytest.mark.parametrize("batch,pinned", [(500, False), (5003, True), (9000, False)])
def test_host_buffer_entry_point(batch, pinned):
    """toom_mul_batched_host (bench.py's e2e path): host buffers in and out,
    chunks pipelined over streams (copies overlap the kernels), ragged last
    chunk; pinned and pageable buffers."""
    u, v = synth.config_inputs(2, batch=batch, first=777)
    if pinned:
        hu, hv = torch.from_numpy(u).pin_memory(), torch.from_numpy(v).pin_memory()
        hw = torch.empty((batch, 512), dtype=torch.uint32).pin_memory()
        tg.toom_mul_batched_host(hu, hv, B=4, t4=32, t3=32, out=hw)
        w = hw.numpy()
    else:
        w = tg.toom_mul_batched_host(u, v, B=4, t4=32, t3=32)
    idx = np.unique(np.concatenate([[0, batch - 1], np.random.default_rng(batch).integers(0, batch, 120)]))
    assert np.array_equal(w[idx], oracle.toom_batched(u[idx], v[idx], top_B=4, threads=8))


def test_workspace_user_provided():
    """toom_set_workspace: a caller-owned buffer is used (and a too-small one
    is an error, not a silent reallocation)."""
    u, v = synth.config_inputs(2, batch=300)
    need = tg.workspace_bytes(256, 300, B=4, t4=32, t3=32)
    buf = torch.empty(need // 4 + 64, dtype=torch.int32, device="cuda")
    try:
        tg.lib().toom_set_workspace(buf.data_ptr(), buf.numel() * 4)
        w = run_batched(u, v, 4, t4=32, t3=32)
        assert np.array_equal(w, oracle.toom_batched(u, v, top_B=4, threads=8))
        tg.lib().toom_set_workspace(buf.data_ptr(), 1024)
        with pytest.raises(tg.ToomError) as ei:
            run_batched(u, v, 4, t4=32, t3=32)
        assert ei.value.status == tg.TOOM_ENOMEM
    finally:
        tg.lib().toom_set_workspace(None, 0)
    assert np.array_equal(run_batched(u, v, 4, t4=32, t3=32), oracle.toom_batched(u, v, top_B=4, threads=8))


def test_streams_and_repeat_determinism():
    """The same call on a side stream and repeated calls give identical
    limbs (positional results; no schedule dependence)."""
    u, v = synth.config_inputs(3, batch=64, first=3000)
    a = run_batched(u, v, 8)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        w = tg.toom_mul_batched(dev(u), dev(v), B=8, stream=s)
    s.synchronize()
    assert np.array_equal(a, host(w))
    assert np.array_equal(a, run_batched(u, v, 8))


@pytest.mark.parametrize("n", [1 << 13, 20011, 1 << 16])
def test_t16_matrix_form_equals_newton_program(n):
    """The matrix-form Toom-16 interpolation (f1) against the
    staged Newton program and the oracle, through
    toom_mul and through the stage export (the sharded C5 top level)."""
    seed = synth.seed_for(5)
    u = synth.uniform_limbs(seed, 21, 1, 0, n)[0]
    v = synth.uniform_limbs(seed, 21, 1, 1, n)[0]
    u[: n // 3] = 0xFFFFFFFF          # long carry runs
    got = {}
    try:
        for mode in (True, False):
            tg.set_t16_matrix(mode)
            got[mode] = host(tg.toom_mul(dev(u), dev(v), B=16))
            U, V = tg.eval_points(dev(u[None]), 16), tg.eval_points(dev(v[None]), 16)
            Y = tg.mul_signed_batched(U[:, 0].contiguous(), V[:, 0].contiguous(), B=4)
            got[(mode, "stage")] = host(tg.interp_recompose(Y.view(31, 1, -1).contiguous(), n, 16))[0]
    finally:
        tg.set_t16_matrix(True)
    want = oracle.schoolbook(u, v) if n <= 20011 else oracle.toom(u, v, top_B=16)
    for k, w in got.items():
        assert np.array_equal(w, want), k


# ------------------------------------------------------------ squaring


@pytest.mark.parametrize("B,n,kw,batch", [(4, 256, dict(t4=32, t3=32), 3000), (3, 96, dict(t4=10**9, t3=10**9), 260),
                                          (8, 2048, {}, 64), (4, 1000, {}, 50), (3, 300, dict(t4=64, t3=64), 77),
                                          (4, 250, dict(t4=32, t3=32), 99)])
def test_squaring_batched(B, n, kw, batch):
    """toom_sqr_batched (one evaluation per level, squaring base case) against
    the oracle's schoolbook u*u, with all-ones and negative-point cases."""
    rng = np.random.default_rng(n * 11 + B)
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    u[1] = 0
    u[2, 1::2] = 0xFFFFFFFF
    u[2, ::2] = 0
    w = host(tg.toom_sqr_batched(dev(u), B=B, **kw))
    assert np.array_equal(w, oracle.schoolbook_batched(u, u))
    # and the plain multiply of u by a copy of u agrees
    w2 = run_batched(u, u.copy(), B, **kw)
    assert np.array_equal(w, w2)


@pytest.mark.parametrize("B,n", [(4, 20000), (16, 9000), (4, 4100)])
def test_squaring_long_path(B, n):
    """toom_mul(a, a): the long-vector and instance-resident levels evaluate
    once; result equal to the schoolbook square."""
    rng = np.random.default_rng(n + B)
    a = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    a[: n // 4] = 0xFFFFFFFF
    da = dev(a)
    w = host(tg.toom_mul(da, da, B=B))
    assert np.array_equal(w, oracle.schoolbook(a, a))


def test_squaring_c3_square_classes():
    """C3's all-ones and alternating quarters are squares (u = v): the
    squaring path gives their closed forms."""
    u, _ = synth.config_inputs(3)
    sub = np.concatenate([u[0:64], u[1024:1088]])
    w = host(tg.toom_sqr_batched(dev(sub), B=8))
    N = 65536
    ones = synth.from_int((1 << (2 * N)) - (1 << (N + 1)) + 1, 4096)
    assert (w[:64] == ones[None, :]).all()
    alt = synth.to_int(u[1024])
    assert (w[64:] == synth.from_int(alt * alt, 4096)[None, :]).all()


# ------------------------------------------------------------ B = 32


@pytest.mark.parametrize("n", [700, 5000, 40000])
def test_b32_paper_points_long_path(n):
    """B = 32 with the paper's points 0, +-2^j, j < 31 (the
    64-bit CPU code allows B = 32): divisors up to 2^60 run as 2-adic divisions
    by their 32-bit word factors on 32-bit limbs.  Bit-exact against the
    schoolbook, including all-ones operands (long carry chains)."""
    rng = np.random.default_rng(n)
    a = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    info = tg.plan_describe(n, 1, B=32)
    assert info["levels"][0]["B"] == 32 and info["levels"][0]["npts"] == 63 and info["levels"][0]["long"]
    w = host(tg.toom_mul(dev(a), dev(b), B=32))
    assert np.array_equal(w, oracle.schoolbook(a, b))
    ones = np.full(n, 0xFFFFFFFF, np.uint32)
    w = host(tg.toom_mul(dev(ones), dev(b), B=32))
    assert np.array_equal(w, oracle.schoolbook(ones, b))


def test_b32_stage_exports():
    n = 3000
    rng = np.random.default_rng(32)
    u = rng.integers(0, 2**32, (1, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (1, n), dtype=np.uint64).astype(np.uint32)
    U, V = tg.eval_points(dev(u), 32), tg.eval_points(dev(v), 32)
    assert U.shape[0] == 63
    Y = tg.mul_signed_batched(U[:, 0].contiguous(), V[:, 0].contiguous(), B=4)
    w = host(tg.interp_recompose(Y.view(63, 1, -1).contiguous(), n, 32))
    assert np.array_equal(w[0], oracle.schoolbook(u[0], v[0]))


# ------------------------------------------------------------ NTT inner multiplier (§5)


@pytest.mark.parametrize("nu,nv", [(700, 700), (5000, 3001), (1 << 15, 1 << 15)])
def test_ntt_inner_multiplier(nu, nv):
    rng = np.random.default_rng(nu + nv)
    a = rng.integers(0, 2**32, nu, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, nv, dtype=np.uint64).astype(np.uint32)
    a[: nu // 5] = 0xFFFFFFFF
    w = host(tg.toom_mul_ntt(dev(a), dev(b), B=0))
    assert np.array_equal(w, oracle.schoolbook(a, b))


@pytest.mark.parametrize("B,n", [(16, 20011), (4, 9000), (3, 5000), (16, 1 << 16)])
def test_toom_wrapper_over_ntt(B, n):
    """Toom-B top level (long path) with its 2B-1 signed pointwise products by
    the NTT: bit-exact against the oracle."""
    seed = synth.seed_for(5)
    u = synth.uniform_limbs(seed, 31, 1, 0, n)[0]
    v = synth.uniform_limbs(seed, 31, 1, 1, n)[0]
    v[n // 2:] = 0xFFFFFFFF
    w = host(tg.toom_mul_ntt(dev(u), dev(v), B=B))
    want = oracle.schoolbook(u, v) if n <= 20011 else oracle.toom(u, v, top_B=16)
    assert np.array_equal(w, want)
    check_residues(u, v, w)
