// Number-theoretic-transform inner multiplier for the Toom top-level wrapper
// (§5: Toom-Cook "as a top-level wrapper
// around" a different multiplication algorithm -- the paper wraps GMP's FFT;
// here the 2B-1 pointwise products of a long-vector top level run through an
// exact NTT over the prime p = 2^64 - 2^32 + 1).
//
// A product of two non-negative values of e limbs: both are split into 16-bit
// digits (2e digits, zero-padded to N >= 4e), transformed (decimation in
// frequency, natural order in, bit-reversed out), multiplied pointwise (times
// N^-1), transformed back (decimation in time, bit-reversed in, natural out);
// coefficient k of the digit convolution is < 2e * 2^32 <= 2^53 < p, so the
// residues ARE the coefficients, and w = sum_k c_k 2^(16 k) is formed by one
// carry-resolving long op (longvec2.cuh) over the coefficient words.
// Signed (two's-complement) evaluated values are multiplied as magnitudes and
// the product negated when the signs differ.
#pragma once

namespace tg {

constexpr uint64_t NTT_P = 0xFFFFFFFF00000001ull;   // 2^64 - 2^32 + 1
constexpr uint64_t NTT_G = 7;                        // generator of the multiplicative group

__host__ __device__ __forceinline__ uint64_t gl_add(uint64_t a, uint64_t b) {
    uint64_t s = a + b;
    // s < a: wrapped past 2^64 = 2^32 - 1 (mod p)
    if (s < a) s += 0xFFFFFFFFull;
    if (s >= NTT_P) s -= NTT_P;
    return s;
}
__host__ __device__ __forceinline__ uint64_t gl_sub(uint64_t a, uint64_t b) {
    uint64_t d = a - b;
    if (a < b) d -= 0xFFFFFFFFull;   // + p = - (2^32 - 1) (mod 2^64)
    return d;
}
// 128-bit x = hi 2^64 + lo -> x mod p, with 2^64 = 2^32 - 1 and 2^96 = -1 (mod p)
__host__ __device__ __forceinline__ uint64_t gl_reduce(uint64_t lo, uint64_t hi) {
    const uint64_t hh = hi >> 32, hl = hi & 0xFFFFFFFFull;
    uint64_t t = lo - hh;                       // lo - hh * 2^96 -> lo - hh
    if (lo < hh) t -= 0xFFFFFFFFull;            // borrow: + p
    const uint64_t m = (hl << 32) - hl;         // hl * (2^32 - 1)
    uint64_t r = t + m;
    if (r < t) r += 0xFFFFFFFFull;
    if (r >= NTT_P) r -= NTT_P;
    return r;
}
__host__ __device__ __forceinline__ uint64_t gl_mul(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
    return gl_reduce(a * b, __umul64hi(a, b));
#else
    const unsigned __int128 x = (unsigned __int128)a * b;
    return gl_reduce((uint64_t)x, (uint64_t)(x >> 64));
#endif
}
__host__ __device__ inline uint64_t gl_pow(uint64_t b, uint64_t e) {
    uint64_t r = 1;
    while (e) {
        if (e & 1) r = gl_mul(r, b);
        b = gl_mul(b, b);
        e >>= 1;
    }
    return r;
}

// 16-bit digits of |a| for a [count][e] two's-complement (sgn) or unsigned
// values: dst [count][N] (digit d of instance c at c*N + d), zero padded.
// |a| = ~a + 1 for negative a: limbs below the lowest nonzero limb z stay 0,
// limb z becomes -a_z, the limbs above ~a_i (z from k_ntt_lowest_nz).
__global__ void k_ntt_digits(const uint32_t* __restrict__ a, long long a_is, int e, int sgn, const int* __restrict__ z,
                             uint64_t* __restrict__ dst, int N) {
    const long long c = blockIdx.y;
    const uint32_t* ai = a + c * a_is;
    const bool neg = sgn && (ai[e - 1] >> 31);
    const int zc = neg ? z[c] : 0;
    for (int d = blockIdx.x * blockDim.x + threadIdx.x; d < N; d += gridDim.x * blockDim.x) {
        const int i = d >> 1;
        uint32_t x = 0;
        if (i < e) {
            x = ai[i];
            if (neg) x = i < zc ? 0u : (i == zc ? 0u - x : ~x);
        }
        dst[c * (long long)N + d] = (d & 1) ? (x >> 16) : (x & 0xFFFFu);
    }
}

// lowest nonzero limb of each instance (e if zero): z[c] = min i with a_i != 0
__global__ void k_ntt_lowest_nz(const uint32_t* __restrict__ a, long long a_is, int e, int* __restrict__ z) {
    const long long c = blockIdx.y;
    const uint32_t* ai = a + c * a_is;
    int best = e;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < e; i += gridDim.x * blockDim.x)
        if (ai[i]) { best = i; break; }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, d));
    if ((threadIdx.x & 31) == 0 && best < e) atomicMin(z + c, best);
}

// decimation-in-frequency stage (half size h): a[j], a[j+h] -> a[j]+a[j+h], (a[j]-a[j+h]) w^j
// over every block of 2h; tw[k] = omega^k (k < N/2), stride N/(2h)
__global__ void k_ntt_dif_stage(uint64_t* __restrict__ a, int N, int h, const uint64_t* __restrict__ tw) {
    const long long c = blockIdx.y;
    uint64_t* x = a + c * (long long)N;
    const int stride = N / (2 * h);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N / 2; t += gridDim.x * blockDim.x) {
        const int blk = t / h, j = t - blk * h;
        const int i0 = blk * 2 * h + j;
        const uint64_t u = x[i0], v = x[i0 + h];
        x[i0] = gl_add(u, v);
        x[i0 + h] = gl_mul(gl_sub(u, v), tw[(long long)j * stride]);
    }
}
// decimation-in-time stage (half size h): a[j+h] *= w^-j, then the butterfly
__global__ void k_ntt_dit_stage(uint64_t* __restrict__ a, int N, int h, const uint64_t* __restrict__ twi) {
    const long long c = blockIdx.y;
    uint64_t* x = a + c * (long long)N;
    const int stride = N / (2 * h);
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N / 2; t += gridDim.x * blockDim.x) {
        const int blk = t / h, j = t - blk * h;
        const int i0 = blk * 2 * h + j;
        const uint64_t u = x[i0], v = gl_mul(x[i0 + h], twi[(long long)j * stride]);
        x[i0] = gl_add(u, v);
        x[i0 + h] = gl_sub(u, v);
    }
}

// three stages (half sizes h = 4q, 2q, q) on the 8 elements x_k = a[base + k q]
// of one residue class j0 (mod q) of a block of 2h, in registers
__host__ __device__ __forceinline__ void ntt_dif_r8(uint64_t (&x)[8], int j0, int q, int N, const uint64_t* tw) {
    const long long s4 = N / (8ll * q), s2 = N / (4ll * q), s1 = N / (2ll * q);
#pragma unroll
    for (int k = 0; k < 4; ++k) {   // half size 4q
        const uint64_t u = x[k], v = x[k + 4];
        x[k] = gl_add(u, v);
        x[k + 4] = gl_mul(gl_sub(u, v), tw[(long long)(j0 + k * q) * s4]);
    }
#pragma unroll
    for (int g = 0; g < 8; g += 4)  // half size 2q
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint64_t u = x[g + k], v = x[g + k + 2];
            x[g + k] = gl_add(u, v);
            x[g + k + 2] = gl_mul(gl_sub(u, v), tw[(long long)(j0 + k * q) * s2]);
        }
    const uint64_t t1 = tw[(long long)j0 * s1];
#pragma unroll
    for (int k = 0; k < 8; k += 2) {  // half size q
        const uint64_t u = x[k], v = x[k + 1];
        x[k] = gl_add(u, v);
        x[k + 1] = gl_mul(gl_sub(u, v), t1);
    }
}
// the inverse: half sizes q, 2q, 4q (decimation in time)
__host__ __device__ __forceinline__ void ntt_dit_r8(uint64_t (&x)[8], int j0, int q, int N, const uint64_t* twi) {
    const long long s4 = N / (8ll * q), s2 = N / (4ll * q), s1 = N / (2ll * q);
    const uint64_t t1 = twi[(long long)j0 * s1];
#pragma unroll
    for (int k = 0; k < 8; k += 2) {
        const uint64_t u = x[k], v = gl_mul(x[k + 1], t1);
        x[k] = gl_add(u, v);
        x[k + 1] = gl_sub(u, v);
    }
#pragma unroll
    for (int g = 0; g < 8; g += 4)
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const uint64_t u = x[g + k], v = gl_mul(x[g + k + 2], twi[(long long)(j0 + k * q) * s2]);
            x[g + k] = gl_add(u, v);
            x[g + k + 2] = gl_sub(u, v);
        }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint64_t u = x[k], v = gl_mul(x[k + 4], twi[(long long)(j0 + k * q) * s4]);
        x[k] = gl_add(u, v);
        x[k + 4] = gl_sub(u, v);
    }
}
// three global stages per pass (half sizes 4q, 2q, q forward; q, 2q, 4q inverse)
template <bool INV>
__global__ void __launch_bounds__(256) k_ntt_r8(uint64_t* __restrict__ a, int N, int q, const uint64_t* __restrict__ tw) {
    const long long c = blockIdx.y;
    uint64_t* xa = a + c * (long long)N;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < N / 8; t += gridDim.x * blockDim.x) {
        const int blk = t / q, j0 = t - blk * q;
        const long long base = (long long)blk * 8 * q + j0;
        uint64_t x[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = xa[base + (long long)k * q];
        if (INV) ntt_dit_r8(x, j0, q, N, tw);
        else ntt_dif_r8(x, j0, q, N, tw);
#pragma unroll
        for (int k = 0; k < 8; ++k) xa[base + (long long)k * q] = x[k];
    }
}

// the small stages in shared memory: a CTA owns one block of NTT_SB
// consecutive elements and runs every stage with h < NTT_SB
constexpr int NTT_SB = 2048;
__global__ void __launch_bounds__(512) k_ntt_dif_tail(uint64_t* __restrict__ a, int N, const uint64_t* __restrict__ tw) {
    __shared__ uint64_t s[NTT_SB];
    const long long c = blockIdx.y;
    uint64_t* x = a + c * (long long)N + (long long)blockIdx.x * NTT_SB;
    for (int i = threadIdx.x; i < NTT_SB; i += blockDim.x) s[i] = x[i];
    __syncthreads();
    for (int h = NTT_SB / 2; h >= 1; h >>= 1) {
        const int stride = N / (2 * h);
        for (int t = threadIdx.x; t < NTT_SB / 2; t += blockDim.x) {
            const int blk = t / h, j = t - blk * h;
            const int i0 = blk * 2 * h + j;
            const uint64_t u = s[i0], v = s[i0 + h];
            s[i0] = gl_add(u, v);
            s[i0 + h] = gl_mul(gl_sub(u, v), tw[(long long)j * stride]);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < NTT_SB; i += blockDim.x) x[i] = s[i];
}
__global__ void __launch_bounds__(512) k_ntt_dit_head(uint64_t* __restrict__ a, int N, const uint64_t* __restrict__ twi) {
    __shared__ uint64_t s[NTT_SB];
    const long long c = blockIdx.y;
    uint64_t* x = a + c * (long long)N + (long long)blockIdx.x * NTT_SB;
    for (int i = threadIdx.x; i < NTT_SB; i += blockDim.x) s[i] = x[i];
    __syncthreads();
    for (int h = 1; h < NTT_SB; h <<= 1) {
        const int stride = N / (2 * h);
        for (int t = threadIdx.x; t < NTT_SB / 2; t += blockDim.x) {
            const int blk = t / h, j = t - blk * h;
            const int i0 = blk * 2 * h + j;
            const uint64_t u = s[i0], v = gl_mul(s[i0 + h], twi[(long long)j * stride]);
            s[i0] = gl_add(u, v);
            s[i0 + h] = gl_sub(u, v);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < NTT_SB; i += blockDim.x) x[i] = s[i];
}

// a = a * b * N^-1 (pointwise, bit-reversed order on both sides)
__global__ void k_ntt_pointwise(uint64_t* __restrict__ a, const uint64_t* __restrict__ b, long long total, uint64_t ninv) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x)
        a[i] = gl_mul(gl_mul(a[i], b[i]), ninv);
}

// w[c] = -w[c] (two's complement, W limbs) where the operand signs differ:
// limbs below the lowest nonzero limb z stay 0, limb z -> -w_z, above -> ~w_i
__global__ void k_ntt_negate(uint32_t* __restrict__ w, long long w_is, int W, const uint32_t* __restrict__ ua, long long u_is,
                             int ue, const uint32_t* __restrict__ va, long long v_is, int ve, const int* __restrict__ z) {
    const long long c = blockIdx.y;
    const bool neg = ((ua[c * u_is + ue - 1] ^ va[c * v_is + ve - 1]) >> 31) != 0;
    if (!neg) return;
    uint32_t* wi = w + c * w_is;
    const int zc = z[c];
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < W; i += gridDim.x * blockDim.x) {
        if (i < zc) continue;
        wi[i] = i == zc ? 0u - wi[i] : ~wi[i];
    }
}

}  // namespace tg
