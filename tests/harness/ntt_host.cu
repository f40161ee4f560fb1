// Host-side check of the NTT inner multiplier's arithmetic (csrc/ntt.cuh,
// compiled for the host by tests/test_host_ntt.py): Goldilocks add / sub / mul
// against 128-bit reference arithmetic, and the kernels' DIF -> pointwise ->
// DIT sequence (same loop bodies) against a schoolbook digit convolution.
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
namespace tg {}
#include "ntt.cuh"   // -I paper_1602_02740_b200/csrc
using namespace tg;
int main() {
    std::mt19937_64 r(1);
    // mulmod vs __int128
    for (int i = 0; i < 1000000; ++i) {
        uint64_t a = r() % NTT_P, b = r() % NTT_P;
        if (i < 10) { a = NTT_P - 1 - i; b = NTT_P - 1; }
        unsigned __int128 x = (unsigned __int128)a * b;
        uint64_t want = (uint64_t)(x % NTT_P);
        if (gl_mul(a, b) != want) { printf("mul fail %llu %llu\n", (unsigned long long)a, (unsigned long long)b); return 1; }
        uint64_t s = (uint64_t)(((unsigned __int128)a + b) % NTT_P);
        if (gl_add(a, b) != s) { printf("add fail\n"); return 1; }
        uint64_t d = (uint64_t)(((unsigned __int128)a + NTT_P - b) % NTT_P);
        if (gl_sub(a, b) != d) { printf("sub fail\n"); return 1; }
    }
    // DIF forward + DIT inverse = identity * N; convolution check
    const int N = 64;
    uint64_t w = gl_pow(NTT_G, (NTT_P - 1) / N), wi = gl_pow(w, NTT_P - 2);
    std::vector<uint64_t> tw(N / 2), twi(N / 2);
    uint64_t x = 1, y = 1;
    for (int k = 0; k < N / 2; ++k) { tw[k] = x; twi[k] = y; x = gl_mul(x, w); y = gl_mul(y, wi); }
    std::vector<uint64_t> a(N, 0), b(N, 0), c(N, 0);
    for (int i = 0; i < N / 2; ++i) { a[i] = r() & 0xFFFF; b[i] = r() & 0xFFFF; }
    for (int i = 0; i < N; ++i) for (int j = 0; j < N; ++j) if (i + j < N) c[i + j] += a[i] * b[j];
    auto dif = [&](std::vector<uint64_t>& v) {
        for (int h = N / 2; h >= 1; h >>= 1) {
            int stride = N / (2 * h);
            for (int t = 0; t < N / 2; ++t) { int blk = t / h, j = t - blk * h, i0 = blk * 2 * h + j;
                uint64_t u = v[i0], q = v[i0 + h]; v[i0] = gl_add(u, q); v[i0 + h] = gl_mul(gl_sub(u, q), tw[j * stride]); }
        }
    };
    auto dit = [&](std::vector<uint64_t>& v) {
        for (int h = 1; h < N; h <<= 1) {
            int stride = N / (2 * h);
            for (int t = 0; t < N / 2; ++t) { int blk = t / h, j = t - blk * h, i0 = blk * 2 * h + j;
                uint64_t u = v[i0], q = gl_mul(v[i0 + h], twi[j * stride]); v[i0] = gl_add(u, q); v[i0 + h] = gl_sub(u, q); }
        }
    };
    dif(a); dif(b);
    uint64_t ninv = gl_pow(N, NTT_P - 2);
    for (int i = 0; i < N; ++i) a[i] = gl_mul(gl_mul(a[i], b[i]), ninv);
    dit(a);
    for (int i = 0; i < N; ++i) if (a[i] != c[i]) { printf("conv fail at %d: %llu vs %llu\n", i, (unsigned long long)a[i], (unsigned long long)c[i]); return 1; }
    // radix-8 passes (three stages at once, as k_ntt_r8) == three radix-2 stages
    {
        const int M = 1 << 14, SB = 64;
        uint64_t wm = gl_pow(NTT_G, (NTT_P - 1) / M), wmi = gl_pow(wm, NTT_P - 2);
        std::vector<uint64_t> T(M / 2), TI(M / 2);
        uint64_t x1 = 1, y1 = 1;
        for (int k = 0; k < M / 2; ++k) { T[k] = x1; TI[k] = y1; x1 = gl_mul(x1, wm); y1 = gl_mul(y1, wmi); }
        std::vector<uint64_t> v(M), r2, r8;
        for (auto& z : v) z = r() % NTT_P;
        auto st2 = [&](std::vector<uint64_t>& a, int h, bool inv) {
            const int stride = M / (2 * h);
            for (int t = 0; t < M / 2; ++t) { int blk = t / h, j = t - blk * h, i0 = blk * 2 * h + j;
                if (!inv) { uint64_t u = a[i0], q = a[i0 + h]; a[i0] = gl_add(u, q); a[i0 + h] = gl_mul(gl_sub(u, q), T[j * stride]); }
                else { uint64_t u = a[i0], q = gl_mul(a[i0 + h], TI[j * stride]); a[i0] = gl_add(u, q); a[i0 + h] = gl_sub(u, q); } }
        };
        auto st8 = [&](std::vector<uint64_t>& a, int q, bool inv) {
            for (int t = 0; t < M / 8; ++t) { int blk = t / q, j0 = t - blk * q; long long base = (long long)blk * 8 * q + j0;
                uint64_t xx[8]; for (int k = 0; k < 8; ++k) xx[k] = a[base + (long long)k * q];
                if (inv) ntt_dit_r8(xx, j0, q, M, TI.data()); else ntt_dif_r8(xx, j0, q, M, T.data());
                for (int k = 0; k < 8; ++k) a[base + (long long)k * q] = xx[k]; }
        };
        r2 = v; r8 = v;
        for (int h = M / 2; h >= 1; h >>= 1) st2(r2, h, false);
        int h = M / 2;
        for (; h / 4 >= SB; h /= 8) st8(r8, h / 4, false);
        for (; h >= 1; h >>= 1) st2(r8, h, false);
        if (r2 != r8) { printf("r8 forward fail\n"); return 1; }
        std::vector<uint64_t> i2 = r2, i8 = r2;
        for (int hh = 1; hh < M; hh <<= 1) st2(i2, hh, true);
        int nglob = 0; for (int x = SB; x < M; x <<= 1) ++nglob;
        for (int hh = 1; hh < SB; hh <<= 1) st2(i8, hh, true);
        h = SB;
        for (int k = 0; k < nglob % 3; ++k, h <<= 1) st2(i8, h, true);
        for (; h < M; h <<= 3) st8(i8, h, true);
        if (i2 != i8) { printf("r8 inverse fail\n"); return 1; }
        const uint64_t minv = gl_pow(M, NTT_P - 2);
        for (int k = 0; k < M; ++k) if (gl_mul(i8[k], minv) != v[k]) { printf("roundtrip fail\n"); return 1; }
    }
    printf("ntt host ok\n");
}
