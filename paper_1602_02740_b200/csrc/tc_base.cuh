// the base case (step a3, y = U(x_k) V(x_k) of E-limb
// operands) as an exact int8 tensor-core product on tcgen05 (UTCIMMA), kept
// beside the IMAD.WIDE.U32 path (k_base) to measure which one wins
// (north_star: tensor cores "only if ... shown by ncu to beat the integer-MAD
// path").  The paper is silent on the base case (§6: "C++ and
// assembler"), so this is an implementation choice, not a reading.
//
// Formulation.  |u|, |v| as L = 4E little-endian bytes.  v is cut into NC =
// ceil(L/32) chunks of K = 32 bytes; with
//     A[m][kk] = u[m - 31 + kk]            (Toeplitz window, 0 outside [0, L))
//     B[kk][c] = v[32 c + 31 - kk]         (chunk c reversed)
// the MMA D = A B gives D[m][c] = sum_{i + j = m + 32 c, j in chunk c} u_i v_j,
// the coefficient of 2^(8 (m + 32 c)) of u * (chunk c of v).  One
// tcgen05.mma.cta_group::1.kind::i8 (M = 128 >= L + 31, N = 16 >= NC,
// K = 32, u8 x u8 -> s32, accumulator in TMEM) per product; every partial sum
// is < 32 * 255^2 < 2^21, so the s32 accumulation is exact.  The epilogue
// reads D back (tcgen05.ld), sums the byte columns S[P] = sum_c D[P - 32c][c]
// and carries them into 2E limbs.
//
// Cost model (why it loses at these sizes): each product needs its own
// Toeplitz A (128 x 32 bytes written to shared memory) because no operand is
// shared between the products of a batch, and the MMA does 128*16*32 = 65536
// byte MACs for E^2 = 324 limb products (E = 18).
#pragma once

namespace tg {

// shared-memory matrix descriptor, K-major, no swizzle (canonical layout
// ((8, m), 2) : ((16 B, SBO), LBO) in 16-byte units; version 1 = sm_100)
__device__ __forceinline__ uint64_t tc_sdesc(uint32_t start, uint32_t lbo, uint32_t sbo) {
    uint64_t d = (uint64_t)((start >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;   // base offset 0, legacy LBO mode, layout type 0 (SWIZZLE_NONE)
}
// instruction descriptor: D s32 (c_format 2), A u8, B u8 (formats 0), K-major,
// N >> 3 at bit 17, M >> 4 at bit 24
__host__ __device__ constexpr uint32_t tc_idesc_i8(int M, int N) {
    return (2u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

constexpr int TC_M = 128, TC_N = 16;
constexpr uint32_t TC_A_SBO = 128, TC_A_LBO = 16 * 128;   // A: 16 row groups per K half
constexpr uint32_t TC_B_SBO = 128, TC_B_LBO = 2 * 128;    // B: 2 row groups per K half

// batched signed base case, interleaved operands [E][count] -> [2E][count]
// (the contract of k_base); one CTA of 128 threads per product at a time
template <int E>
__global__ void __launch_bounds__(128) k_base_tc(const uint32_t* __restrict__ U, const uint32_t* __restrict__ V,
                                                 uint32_t* __restrict__ P, size_t count) {
    constexpr int L = 4 * E, NC = (L + 31) / 32, W = 2 * E;
    static_assert(L + 31 <= TC_M && NC <= TC_N, "E too large for one M = 128 MMA");
    __shared__ __align__(1024) uint8_t As[TC_M * 32];
    __shared__ __align__(1024) uint8_t Bs[TC_N * 32];
    constexpr int UW = E + 48;                       // u words: 8 zero words, u, zeros (rows up to m = 127)
    __shared__ uint32_t Ub[UW];
    __shared__ uint32_t Vb[E + 8];
    __shared__ int Cs[NC][TC_M];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tslot;
    __shared__ uint32_t s_neg;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        mbar_init(&mbar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    for (int i = tid; i < UW; i += blockDim.x) Ub[i] = 0u;
    for (int i = tid; i < E + 8; i += blockDim.x) Vb[i] = 0u;
    for (int i = tid; i < TC_N * 32 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(Bs)[i] = 0u;
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = tslot;
    const uint64_t adesc = tc_sdesc(smem_u32(As), TC_A_LBO, TC_A_SBO);
    const uint64_t bdesc = tc_sdesc(smem_u32(Bs), TC_B_LBO, TC_B_SBO);
    constexpr uint32_t idesc = tc_idesc_i8(TC_M, TC_N);
    unsigned phase = 0;
    for (size_t c = blockIdx.x; c < count; c += gridDim.x) {
        // magnitudes (two's complement -> |x|), one thread per operand
        if (tid == 0 || tid == 32) {
            const uint32_t* src = (tid ? V : U) + c;
            uint32_t* dst = tid ? Vb : Ub + 8;
            const uint32_t neg = __ldg(src + (size_t)(E - 1) * count) >> 31, mask = 0u - neg;
            uint32_t cy = neg;
            for (int i = 0; i < E; ++i) {
                const uint32_t x = (__ldg(src + (size_t)i * count) ^ mask) + cy;
                cy = (x < cy) ? 1u : 0u;
                dst[i] = x;
            }
            if (tid == 0) s_neg = neg;
        }
        __syncthreads();
        const uint32_t neg = s_neg ^ (__ldg(V + (size_t)(E - 1) * count + c) >> 31);
        // A row m = tid: bytes u[m-31 .. m] = padded bytes [m+1, m+33)
        {
            const int sb = tid + 1, w0 = sb >> 2, sh = 8 * (sb & 3);
            uint32_t o[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = __funnelshift_r(Ub[w0 + q], Ub[w0 + q + 1], sh);
            uint8_t* row = As + (tid >> 3) * TC_A_SBO + (tid & 7) * 16;
            *reinterpret_cast<uint4*>(row) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(row + TC_A_LBO) = make_uint4(o[4], o[5], o[6], o[7]);
        }
        // B row n < NC: v[32n + 31 - kk] (chunk n reversed)
        if (tid < NC) {
            const int n = tid;
            uint32_t o[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) o[q] = __byte_perm(Vb[8 * n + 7 - q], 0u, 0x0123);
            uint8_t* row = Bs + (n >> 3) * TC_B_SBO + (n & 7) * 16;
            *reinterpret_cast<uint4*>(row) = make_uint4(o[0], o[1], o[2], o[3]);
            *reinterpret_cast<uint4*>(row + TC_B_LBO) = make_uint4(o[4], o[5], o[6], o[7]);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic smem writes -> async proxy
        __syncthreads();
        if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, {%5, %6, %7, %8}, p;\n\t}\n" ::"r"(tmem),
                "l"(adesc), "l"(bdesc), "r"(idesc), "r"(0), "r"(0), "r"(0), "r"(0), "r"(0));
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             smem_u32(&mbar))
                         : "memory");
        }
        mbar_wait(&mbar, phase);
        phase ^= 1u;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        {
            uint32_t d0, d1, d2, d3;
            const uint32_t ta = tmem + ((uint32_t)(warp * 32) << 16);
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(d0), "=r"(d1), "=r"(d2), "=r"(d3)
                         : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
            const uint32_t d[4] = {d0, d1, d2, d3};
#pragma unroll
            for (int q = 0; q < NC; ++q) Cs[q][tid] = (int)d[q];
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        __syncthreads();
        // limb t = sum_{q<4} S[4t+q] 2^(8q), S[P] = sum_c D[P - 32c][c]
        if (tid < 32) {
            // two limbs per lane (W <= 48 < 64), then a serial carry pass in lane 0
            uint64_t part[2] = {0, 0};
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int t = tid + 32 * h;
                if (t < W) {
                    uint64_t acc = 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const int Pq = 4 * t + q;
                        uint64_t s = 0;
#pragma unroll
                        for (int cc = 0; cc < NC; ++cc) {
                            const int m = Pq - 32 * cc;
                            if (m >= 0 && m < TC_M) s += (uint32_t)Cs[cc][m];
                        }
                        acc += s << (8 * q);
                    }
                    part[h] = acc;
                }
            }
            // carries (lane order), the sign, interleaved stores
            uint64_t cy = 0;
            uint32_t ncy = neg;
            const uint32_t mask = 0u - neg;
            for (int t = 0; t < W; ++t) {
                const uint64_t pt = __shfl_sync(0xffffffffu, t < 32 ? part[0] : part[1], t & 31);
                const uint64_t x = pt + cy;
                cy = x >> 32;
                const uint32_t lo = ((uint32_t)x ^ mask) + ncy;
                ncy = (lo < ncy) ? 1u : 0u;
                if (tid == 0) P[(size_t)t * count + c] = lo;
            }
        }
        __syncthreads();   // Ub / Vb / As / Bs / Cs reuse
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

}  // namespace tg
