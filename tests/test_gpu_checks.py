"""GPU tests of the failure-detection subsystem and of
the boundary's memory contract: the device exact-division check
(TOOM_EINEXACT, "the divisions are exact"), the
residue verification (TOOM_EVERIFY), fault injection, per-stream
workspaces, misaligned pointers and caller workspaces for every plan.
"""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu

tg = pytest.importorskip("paper_1602_02740_b200")


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


@pytest.fixture(autouse=True)
def _reset():
    if not torch.cuda.is_available():
        pytest.fail("no CUDA device: GPU tests must run on the B200 box")
    tg.lib()
    tg.last_error()          # a status left by an earlier test (e.g. an expected TOOM_ENOMEM)
    yield
    tg.debug_fault(0)
    tg.set_check(True)       # read back (and clear) any device flag, then switch off
    tg.last_error()
    tg.set_check(False)
    tg.set_verify(False)
    tg.last_error()


# shapes that exercise every kernel with a checked division: the fused bottom
# rows (T3, T4), the top-level smem rows (C2 top), the row-parallel Toom-8
# top level (C3), the row-parallel lower levels (k_interp_rows_w)
CHECK_CASES = [
    (4, 256, dict(t4=32, t3=32), 2000),        # C2 shape
    (3, 96, dict(t4=10**9, t3=10**9), 300),    # C1 shape
    (8, 2048, {}, 40),                         # C3 shape
    (4, 1026, {}, 60),                         # signed lower levels (rows_w + fused T3)
    (4, 4100, {}, 9),
]


@pytest.mark.parametrize("B,n,kw,batch", CHECK_CASES)
def test_exact_division_check_clean_on_valid_data(B, n, kw, batch):
    rng = np.random.default_rng(n + B)
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    u[0] = 0xFFFFFFFF
    v[0] = 0xFFFFFFFF
    u[1] = 0
    u[2, 1::2] = 0xFFFFFFFF
    u[2, ::2] = 0
    v[2] = u[2]
    tg.set_check(True)
    tg.set_verify(True)
    assert tg.last_error() == tg.TOOM_OK     # clean start
    w = tg.toom_mul_batched(dev(u), dev(v), B=B, **kw)
    assert tg.last_error() == tg.TOOM_OK
    assert np.array_equal(host(w), oracle.schoolbook_batched(u, v))


def test_fault_injection_reports_inexact_division():
    u, v = synth.config_inputs(2, batch=256)
    tg.set_check(True)
    tg.last_error()
    tg.debug_fault(1)
    w = tg.toom_mul_batched(dev(u), dev(v), B=4, t4=32, t3=32)
    st = tg.last_error()
    assert st == tg.TOOM_EINEXACT
    # the fault really changed a product
    assert not np.array_equal(host(w), oracle.schoolbook_batched(u, v))
    tg.debug_fault(0)
    tg.toom_mul_batched(dev(u), dev(v), B=4, t4=32, t3=32)
    assert tg.last_error() == tg.TOOM_OK


@pytest.mark.parametrize("mode", [0, 1])
def test_fault_injection_other_c2_modes(mode):
    """The per-row C2 bottom (modes 0, 1) flips a product bit; its own row
    divisions catch it."""
    u, v = synth.config_inputs(2, batch=256)
    tg.set_c2_mode(mode)
    try:
        tg.set_check(True)
        tg.last_error()
        tg.debug_fault(1)
        tg.toom_mul_batched(dev(u), dev(v), B=4, t4=32, t3=32)
        assert tg.last_error() == tg.TOOM_EINEXACT
    finally:
        tg.debug_fault(0)
        tg.set_c2_mode(2)


def test_c2_top_serial_carry_chain_equals_oracle():
    """The C2 top level's rare path (csrc/toplevel_cls.cuh phase 3: a carry
    that wraps a segment's limb 0 sends the product through the serial
    carry/borrow chain) forced for every product (debug kind 2)."""
    u, v = synth.config_inputs(2, batch=1000, first=7)
    u[:4] = 0xFFFFFFFF
    try:
        tg.debug_fault(2)
        w = host(tg.toom_mul_batched(dev(u), dev(v), B=4, t4=32, t3=32))
    finally:
        tg.debug_fault(0)
    assert np.array_equal(w, oracle.schoolbook_batched(u, v))


def test_fault_injection_caught_by_verify_alone():
    u, v = synth.config_inputs(2, batch=256)
    tg.set_verify(True)
    tg.last_error()
    tg.debug_fault(1)
    tg.toom_mul_batched(dev(u), dev(v), B=4, t4=32, t3=32)
    assert tg.last_error() == tg.TOOM_EVERIFY


def test_verify_catches_corrupted_result_via_toom_mul():
    """verify on the single-product entry point, long path (C4-like shape)."""
    rng = np.random.default_rng(5)
    n = 20000
    a = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    b = rng.integers(0, 2**32, n, dtype=np.uint64).astype(np.uint32)
    tg.set_verify(True)
    tg.last_error()
    w = tg.toom_mul(dev(a), dev(b), B=4)
    assert tg.last_error() == tg.TOOM_OK
    assert np.array_equal(host(w), oracle.schoolbook(a, b))
    w2 = tg.toom_mul(dev(a), dev(b[:-7]), B=16)    # unbalanced, Toom-16 top level
    assert tg.last_error() == tg.TOOM_OK
    assert np.array_equal(host(w2), oracle.schoolbook(a, b[:-7]))


def test_two_unsynchronized_streams_do_not_share_workspace():
    """two calls on two streams with no sync between them must not
    corrupt each other (per-stream workspaces)."""
    ua, va = synth.config_inputs(2, batch=20000, first=0)
    ub, vb = synth.config_inputs(2, batch=20000, first=30000)
    da, db = dev(ua), dev(ub)
    dva, dvb = dev(va), dev(vb)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    for _ in range(3):
        with torch.cuda.stream(s1):
            wa = tg.toom_mul_batched(da, dva, B=4, t4=32, t3=32, stream=s1)
        with torch.cuda.stream(s2):
            wb = tg.toom_mul_batched(db, dvb, B=4, t4=32, t3=32, stream=s2)
    torch.cuda.synchronize()
    idx = np.arange(0, 20000, 97)
    assert np.array_equal(host(wa)[idx], oracle.toom_batched(ua[idx], va[idx], top_B=4, threads=8))
    assert np.array_equal(host(wb)[idx], oracle.toom_batched(ub[idx], vb[idx], top_B=4, threads=8))


def test_caller_workspace_shared_by_two_streams():
    u, v = synth.config_inputs(2, batch=3000)
    need = tg.workspace_bytes(256, 3000, B=4, t4=32, t3=32)
    buf = torch.empty(need // 4 + 64, dtype=torch.int32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    try:
        tg.lib().toom_set_workspace(buf.data_ptr(), buf.numel() * 4)
        du, dv = dev(u), dev(v)
        torch.cuda.synchronize()
        with torch.cuda.stream(s1):
            w1 = tg.toom_mul_batched(du, dv, B=4, t4=32, t3=32, stream=s1)
        with torch.cuda.stream(s2):
            w2 = tg.toom_mul_batched(dv, du, B=4, t4=32, t3=32, stream=s2)
        torch.cuda.synchronize()
    finally:
        tg.lib().toom_set_workspace(None, 0)
    want = oracle.toom_batched(u, v, top_B=4, threads=8)
    assert np.array_equal(host(w1), want)
    assert np.array_equal(host(w2), want)


@pytest.mark.parametrize("n", [1, 7, 33, 64])
def test_workspace_bytes_covers_schoolbook_only_plans(n):
    rng = np.random.default_rng(n)
    batch = 100
    u = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    v = rng.integers(0, 2**32, (batch, n), dtype=np.uint64).astype(np.uint32)
    need = tg.workspace_bytes(n, batch, B=4)
    assert need > 0
    buf = torch.empty(need // 4 + 1, dtype=torch.int32, device="cuda")
    try:
        tg.lib().toom_set_workspace(buf.data_ptr(), need)
        w = tg.toom_mul_batched(dev(u), dev(v), B=4)
        torch.cuda.synchronize()
    finally:
        tg.lib().toom_set_workspace(None, 0)
    assert np.array_equal(host(w), oracle.schoolbook_batched(u, v))


def test_misaligned_operand_and_output_pointers():
    """Views at a 4-byte (not 16-byte) offset: the vectorised staging and
    stores must fall back instead of faulting."""
    u, v = synth.config_inputs(2, batch=500)
    batch, n = u.shape
    bu = torch.zeros(batch * n + 1, dtype=torch.uint32, device="cuda")
    bv = torch.zeros(batch * n + 3, dtype=torch.uint32, device="cuda")
    bw = torch.zeros(batch * 2 * n + 1, dtype=torch.uint32, device="cuda")
    du = bu[1:].view(batch, n)
    dv = bv[3:].view(batch, n)
    dw = bw[1:].view(batch, 2 * n)
    du.copy_(dev(u))
    dv.copy_(dev(v))
    assert du.data_ptr() % 16 and dw.data_ptr() % 16
    tg.toom_mul_batched(du, dv, B=4, t4=32, t3=32, out=dw)
    torch.cuda.synchronize()
    assert np.array_equal(host(dw), oracle.toom_batched(u, v, top_B=4, threads=8))


def test_out_shape_is_validated():
    x = torch.zeros((4, 96), dtype=torch.uint32, device="cuda")
    with pytest.raises(ValueError):
        tg.toom_mul_batched(x, x, B=3, out=torch.empty((4, 191), dtype=torch.uint32, device="cuda"))
    with pytest.raises(ValueError):
        tg.toom_mul(x[0], x[1], B=3, out=torch.empty(100, dtype=torch.uint32, device="cuda"))
    y = torch.zeros((31, 1, 10), dtype=torch.uint32, device="cuda")
    with pytest.raises(ValueError):
        tg.interp_recompose(y, 5000, 16)


def test_eval_top_single_operand_matches_batched_eval():
    """toom_eval_top launches one thread per instance (no duplicate stores)."""
    u, _ = synth.config_inputs(2, batch=64)
    out = host(tg.eval_top(dev(u), 4))
    assert tg.last_launch_count() == 1
    b = 64
    blocks = [[synth.to_int(u[i, k * b:(k + 1) * b]) for k in range(4)] for i in range(3)]
    pts = [(0, 1), (1, 1), (-1, 1), (2, 1), (-2, 1), (1, 2), (1, 0)]
    e = out.shape[0]
    for i in range(3):
        for k, (p, q) in enumerate(pts):
            want = sum(x * p**j * q ** (3 - j) for j, x in enumerate(blocks[i]))
            got = synth.to_int(out[:, k * 64 + i])
            if got >> (32 * e - 1):
                got -= 1 << (32 * e)
            assert got == want
