// Device-side failure detection.
//
// 1. Exact-division check (TOOM_EINEXACT).  Every division on the
//    interpolation path is exact (§3: "the divisions are exact
//    integer divisions").  The 2-adic division q_t = (x_t - beta_t) o^-1 keeps a
//    borrow beta in [0, o); once the dividend X = o 2^s w is fully
//    sign-extended (its signed carry is 0 or -1), X is divisible by o exactly
//    when beta = 0 (X >= 0) or beta = o - 1 (X < 0), and by 2^s exactly when the
//    low s bits of the first quotient limb are zero.  (From o Q = X + beta 2^(32W)
//    with Q = X o^-1 mod 2^(32W): X = -(beta + [X<0]) 2^(32W) (mod o).)
//    Kernels that know where their dividend ends call TG_CHECK_LOW / _END when
//    the check is switched on (toom_set_check); a failure sets bit 0 of
//    tg_err_flags, which toom_last_error() reads back as TOOM_EINEXACT.
// 2. Result verification (TOOM_EVERIFY): w mod p == (u mod p)(v mod p) mod p for
//    the Mersenne prime p = 2^61 - 1 (the ring homomorphism Z -> Z/p), one warp
//    per product, after the multiplication (toom_set_verify).  A failure sets
//    bit 1 of tg_err_flags.
// 3. Fault injection: tg_fault = 1 flips one bit of one base-case
//    product inside the fused bottom kernel, so that the following exact
//    division is no longer exact (tests expect TOOM_EINEXACT / TOOM_EVERIFY).
#pragma once
#include <stdint.h>

namespace tg {
__device__ unsigned tg_err_flags = 0;   // bit 0 inexact division, bit 1 residue mismatch
// switches in constant memory: read-only inside kernels, so the compiler keeps
// them out of the hot loops (as __device__ globals they were reloaded after
// every global store: C3's row kernel 0.89 -> 1.25 ms)
__constant__ int tg_check_on = 0;       // exact-division checks enabled
__constant__ int tg_fault = 0;          // fault injection (tests only)

__device__ __forceinline__ void tg_flag_inexact() { atomicOr(&tg_err_flags, 1u); }

// the low s bits of the first quotient limb must be zero (exact 2^s division)
__device__ __forceinline__ void tg_check_low(uint32_t q0, int s) {
    if (s > 0 && (q0 & ((1u << s) - 1u))) tg_flag_inexact();
}
// end of a dividend X = X_low + acc 2^(32W) (acc: the signed carry past the
// W processed limbs, corrected for sources read modulo 2^(32W): a negative
// source y_k with multiplier A_k adds -A_k; the borrow chain saw X_low only).
// o Q_res = X_low + bor 2^(32W) and Q = X / o fits W limbs, so X is divisible
// by o exactly when bor = acc (acc >= 0) or acc + o (acc < 0), -o <= acc < o.
__device__ __forceinline__ bool tg_exact_end(uint64_t acc, uint32_t bor, uint32_t o) {
    const long long a = (long long)acc;
    if (a < -(long long)o || a >= (long long)o) return false;
    return (long long)bor == (a >= 0 ? a : a + (long long)o);
}
__device__ __forceinline__ void tg_check_end(uint64_t acc, uint32_t bor, uint32_t o) {
    if (!tg_exact_end(acc, bor, o)) tg_flag_inexact();
}
}  // namespace tg

#define TG_CHECK_LOW(q0, s) \
    do { if (tg::tg_check_on) tg::tg_check_low((q0), (s)); } while (0)
#define TG_CHECK_END(acc, bor, o) \
    do { if (tg::tg_check_on) tg::tg_check_end((acc), (bor), (o)); } while (0)
#define TG_CHECK_ENABLED (tg::tg_check_on)

namespace tg {
// ---- result verification mod p = 2^61 - 1 ----------------------------------
constexpr uint64_t TG_M61 = (1ull << 61) - 1;
__device__ __forceinline__ uint64_t m61_fold(unsigned __int128 x) {   // x < 2^122 -> [0, p)
    uint64_t r = ((uint64_t)x & TG_M61) + (uint64_t)(x >> 61);
    r = (r & TG_M61) + (r >> 61);
    return r >= TG_M61 ? r - TG_M61 : r;
}
__device__ __forceinline__ uint64_t m61_add(uint64_t a, uint64_t b) {
    const uint64_t r = a + b;
    return r >= TG_M61 ? r - TG_M61 : r;
}
// residue mod 2^61 - 1 of limbs a[0..n) (sum of a_i 2^(32 i), 2^(32 i) = 2^((32 i) mod 61)),
// one warp; every lane returns the residue
__device__ __forceinline__ uint64_t m61_residue_warp(const uint32_t* __restrict__ a, size_t n, int lane) {
    uint64_t acc = 0;
    unsigned e = (32u * (unsigned)lane) % 61u;
    for (size_t i = lane; i < n; i += 32) {
        acc = m61_add(acc, m61_fold((unsigned __int128)__ldg(a + i) << e));
        e += 48u;            // 32 * 32 = 1024 = 48 (mod 61)
        if (e >= 61u) e -= 61u;
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) acc = m61_add(acc, __shfl_xor_sync(0xffffffffu, acc, d));
    return acc;
}
// one warp per product: w_i mod p == (u_i mod p)(v_i mod p) mod p, else flag bit 1
__global__ void __launch_bounds__(256) k_verify_m61(const uint32_t* __restrict__ u, size_t nu,
                                                    const uint32_t* __restrict__ v, size_t nv,
                                                    const uint32_t* __restrict__ w, size_t batch) {
    const size_t i = ((size_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (i >= batch) return;
    const uint64_t ru = m61_residue_warp(u + i * nu, nu, lane);
    const uint64_t rv = m61_residue_warp(v + i * nv, nv, lane);
    const uint64_t rw = m61_residue_warp(w + i * (nu + nv), nu + nv, lane);
    if (lane == 0 && m61_fold((unsigned __int128)ru * rv) != rw) atomicOr(&tg_err_flags, 2u);
}
}  // namespace tg
