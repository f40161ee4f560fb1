"""Host test (no GPU) of the NTT inner multiplier's modular arithmetic and
transform order (csrc/ntt.cuh): the header is compiled for the
host with nvcc and run; plus the field facts the multiplier relies on."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

P = (1 << 64) - (1 << 32) + 1


def test_goldilocks_field_facts():
    # p is prime (deterministic Miller-Rabin, bases up to 37 suffice < 3.3e24)
    def is_prime(n):
        d, s = n - 1, 0
        while d % 2 == 0:
            d //= 2
            s += 1
        for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
            x = pow(a, d, n)
            if x in (1, n - 1):
                continue
            for _ in range(s - 1):
                x = x * x % n
                if x == n - 1:
                    break
            else:
                return False
        return True
    assert is_prime(P)
    # 7 generates: 7^((p-1)/q) != 1 for every prime q | p - 1 = 2^32 * 3 * 5 * 17 * 257 * 65537
    assert P - 1 == (1 << 32) * 3 * 5 * 17 * 257 * 65537
    for q in (2, 3, 5, 17, 257, 65537):
        assert pow(7, (P - 1) // q, P) != 1
    # reduction identities used by gl_reduce
    assert pow(2, 64, P) == (1 << 32) - 1 and pow(2, 96, P) == P - 1
    # coefficient bound of the C5 products: 2e digits of 16 bits, e = 2^20 + 2
    e = (1 << 20) + 2
    assert 2 * e * (1 << 32) < P


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="needs nvcc")
def test_ntt_host_arithmetic(tmp_path):
    exe = str(tmp_path / "ntt_host")
    subprocess.check_call(["nvcc", "-std=c++17", "-I", os.path.join(ROOT, "paper_1602_02740_b200", "csrc"), "-o", exe,
                           os.path.join(ROOT, "tests", "harness", "ntt_host.cu")])
    out = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0 and "ntt host ok" in out.stdout, out.stdout + out.stderr
