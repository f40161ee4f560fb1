"""Host-logic tests (no GPU) of the CUDA path's build-time pieces:

* gen/toomgen.py derives each evaluation / interpolation program from the
  paper's method and proves it exact symbolically; here the programs are
  re-checked on random data against the block convolution (the definition
  w_k = sum_{i+j=k} u_i v_j, Eq. 1.3), and
* the emitted LSB-first streaming code (delays, register histories, 2-adic
  exact division) is compiled for the HOST from the very header the kernels
  include (tests/harness/stream_harness.cpp) and compared limb-for-limb with
  exact Python integers.  This harness is test-only; the product has no CPU
  path.
"""
import ctypes
import os
import random
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "paper_1602_02740_b200", "gen"))
import toomgen  # noqa: E402

GEN = os.path.join(ROOT, "paper_1602_02740_b200", "csrc", "generated")
HARNESS = os.path.join(ROOT, "tests", "harness", "stream_harness.cpp")

SETS = {"T3": toomgen.pointset_T3(), "T4": toomgen.pointset_T4(), "P8": toomgen.pointset_paper(8)}


@pytest.fixture(scope="module")
def harness(tmp_path_factory):
    from paper_1602_02740_b200.build import generate
    generate()
    so = str(tmp_path_factory.mktemp("h") / "harness.so")
    subprocess.check_call(["g++", "-O1", "-std=c++17", "-shared", "-fPIC", "-I", GEN, "-o", so, HARNESS])
    L = ctypes.CDLL(so)
    P = ctypes.POINTER(ctypes.c_uint32)
    L.harness_run.argtypes = [ctypes.c_char_p, P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, ctypes.c_int]
    L.harness_run.restype = ctypes.c_int
    return L


def twos(x, w):
    return np.frombuffer((x % (1 << (32 * w))).to_bytes(4 * w, "little"), dtype=np.uint32).copy()


def untwos(a):
    w = a.size
    x = int.from_bytes(np.ascontiguousarray(a).tobytes(), "little")
    return x - (1 << (32 * w)) if x >> (32 * w - 1) else x


def run(h, name, vals, win, wout, nout, fill_mode=1):
    inp = np.concatenate([twos(v, win) for v in vals]) if vals else np.zeros(0, np.uint32)
    out = np.zeros(nout * wout, dtype=np.uint32)
    st = h.harness_run(name.encode(), inp.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), len(vals), win,
                       out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32)), wout, fill_mode)
    assert st == 0
    return [untwos(out[j * wout:(j + 1) * wout]) for j in range(nout)]


@pytest.mark.parametrize("name", list(SETS))
def test_programs_exact_symbolic_and_random(name):
    assert toomgen.selfcheck(SETS[name], trials=30, bits=500, seed=3)


def test_31_point_set_reading():
    # SURVEY §8(c) reading 5: 0, inf, 29 smallest-height +-p/q, last +2/5
    ps = toomgen.pointset_T16_31()
    assert len(ps.points) == 31 and len(set(ps.points)) == 31
    assert ps.points[:2] == [(0, 1), (1, 0)] and ps.points[-1] == (2, 5)
    assert toomgen.selfcheck(ps, trials=3, bits=200)


def test_paper_points_all_B():
    # the paper's points 0, +-2^j for every B up to 16
    for B in range(2, 17):
        assert toomgen.selfcheck(toomgen.pointset_paper(B), trials=3, bits=200)


@pytest.mark.parametrize("name", list(SETS))
def test_streaming_eval_matches_definition(harness, name):
    ps = SETS[name]
    rng = random.Random(11)
    n = ps.B - 1
    for b in (1, 2, 5, 17):
        for _ in range(6):
            # blocks 0..B-2 unsigned (b limbs), top block signed
            blocks = [rng.getrandbits(32 * b) for _ in range(ps.B - 1)]
            blocks.append(rng.randrange(-(1 << (32 * b - 1)), 1 << (32 * b - 1)))
            e = b + 3
            got = run(harness, f"tg_eval_{name}", blocks, b, e, ps.npoints, fill_mode=2)
            want = [sum(u * p**k * q ** (n - k) for k, u in enumerate(blocks)) for (p, q) in ps.points]
            assert got == want


@pytest.mark.parametrize("name", list(SETS))
@pytest.mark.parametrize("half", ["", "_even", "_odd"])
def test_streaming_interp_matches_convolution(harness, name, half):
    ps = SETS[name]
    rng = random.Random(12)
    n = ps.B - 1
    for b in (1, 3, 9):
        for trial in range(6):
            U = [rng.randrange(-(1 << (32 * b)), 1 << (32 * b)) for _ in range(ps.B)]
            V = [rng.randrange(-(1 << (32 * b)), 1 << (32 * b)) for _ in range(ps.B)]
            if trial == 0:
                U = [(1 << (32 * b)) - 1] * ps.B   # all-ones blocks: carry stress
                V = list(U)
            Y = [sum(u * p**k * q ** (n - k) for k, u in enumerate(U)) * sum(v * p**k * q ** (n - k) for k, v in enumerate(V))
                 for (p, q) in ps.points]
            ywidth = max(1, max(abs(y) for y in Y).bit_length() // 32 + 2)
            lw = 2 * b + 2
            got = run(harness, f"tg_interp_{name}{half}", Y, ywidth, lw, 2 * n + 1)
            conv = [sum(U[i] * V[k - i] for i in range(ps.B) if 0 <= k - i < ps.B) for k in range(2 * n + 1)]
            for j in range(2 * n + 1):
                if half == "_even" and j % 2:
                    continue
                if half == "_odd" and j % 2 == 0:
                    continue
                assert got[j] == conv[j], (name, half, b, j)


def test_constexpr_eval_coefficients_match_table(tmp_path):
    """k_eval_top_v4 takes its point coefficients from the generated constexpr
    function tg_evalc_cx_*; they must equal the tg_evalc_* table (the fused
    kernel's) and the homogeneous-point definition p^j q^(n-j) (§2)."""
    from paper_1602_02740_b200.build import generate
    generate()
    src = tmp_path / "cx.cpp"
    src.write_text('#include "toom_programs.cuh"\n#include <cstdio>\n'
                   'int main() {\n'
                   '  for (int k = 0; k < 5; ++k) for (int j = 0; j < 3; ++j)\n'
                   '    std::printf("T3 %d %d %lld %lld\\n", k, j, tg_evalc_cx_T3(k, j), tg_evalc_T3[k][j]);\n'
                   '  for (int k = 0; k < 7; ++k) for (int j = 0; j < 4; ++j)\n'
                   '    std::printf("T4 %d %d %lld %lld\\n", k, j, tg_evalc_cx_T4(k, j), tg_evalc_T4[k][j]);\n'
                   '  static_assert(tg_evalc_cx_T4(3, 3) == 8, "compile-time");\n'
                   '  return 0;\n}\n')
    exe = tmp_path / "cx"
    subprocess.check_call(["g++", "-std=c++17", "-I", GEN, "-o", str(exe), str(src)])
    out = subprocess.check_output([str(exe)], text=True).split("\n")
    rows = [l.split() for l in out if l]
    assert len(rows) == 15 + 28
    for name, k, j, cx, tab in rows:
        ps = SETS[name]
        p, q = ps.points[int(k)]
        want = p ** int(j) * q ** (ps.n - int(j))
        assert int(cx) == int(tab) == want, (name, k, j, cx, tab, want)
