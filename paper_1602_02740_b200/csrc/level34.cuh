// Instance-resident Toom-3/4 levels ("levels at or below
// ~1K limbs must live in SMEM"; here up to ~4K limbs): one CTA per instance
// holds the whole instance in shared memory, so the carries and the exact-
// division borrows of a level resolve with CTA-wide scans and nothing waits
// on another CTA.  Used for the recursion levels between the limb-parallel
// long levels (few, very long operands) and the fused bottom level: C4/C5
// levels with 258..4098-limb operands.
//
//   k_res_eval<B>    step a1 + a2: the parent (row-major, two's complement or
//                    unsigned at the top) staged in smem; each of the 2B-1
//                    points U(p:q) = sum_j p^j q^(B-1-j) u_j (Eq. 1.1-1.2,
//                    homogeneous) formed limb by limb and carry-normalised
//                    (one CTA scan per round of NT x CH limbs), written
//                    row-major (child k of parent c at (k count + c) e).
//   k_res_interp<B>  steps a4 + a5: the 2B-1 child products staged in smem;
//                    the interior coefficients w_j = (sum_k A_jk y_k) / (o_j 2^s_j)
//                    (the even-odd + listing program composed per row,
//                    PAPER.md:162; exact 2-adic division, ref [4]) formed in
//                    smem; then the recomposition w = sum_j w_j 2^(32 b j)
//                    (Eq. 1.3) written to the parent's product.
// Scans: a thread's CH positions are normalised locally; its carry map (3-
// piece, longvec.cuh) and its residue sum lin_p 2^(32 p) mod o are combined
// by warp shuffles and the warps' aggregates; the borrow of position p
// follows from the closed form beta_p = (c_p - 2^(-32 p) sum_{i<p} lin_i 2^(32 i))
// mod o (longvec2.cuh), so a round needs one pass.
#pragma once

namespace tg {

constexpr int RES_CH = 9;        // positions per thread per round (odd: conflict-free smem strides)
constexpr int RES_MAXW = 8;      // warps per CTA

struct ResSmem {
    LCMap wmap[RES_MAXW];
    uint32_t wres[RES_MAXW];
    long long cin;               // state at the start of the current round
    uint32_t bin;
    long long cout;              // state at the end of the round (written by the last thread)
    uint32_t bout;
};

// Mch^tid mod o (forward) and mi^tid (inverse), mi = Mch^-1: warp product scans
__device__ __forceinline__ uint32_t res_pow_tid(uint32_t base, const LMod& M, int lane, int warp) {
    uint32_t pw = base;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const uint32_t t = __shfl_up_sync(0xffffffffu, pw, d);
        if (lane >= d) pw = lv_mulmod(pw, t, M);
    }
    const uint32_t m32 = __shfl_sync(0xffffffffu, pw, 31);
    pw = __shfl_up_sync(0xffffffffu, pw, 1);
    if (lane == 0) pw = 1u % M.o;
    uint32_t wb = 1u % M.o;
    for (int w = 0; w < warp; ++w) wb = lv_mulmod(wb, m32, M);
    return lv_mulmod(pw, wb, M);
}

// per-modulus constants of a round (o = 1: no division)
struct ResDiv {
    uint32_t o, oinv, p32, Mch, mi;
    unsigned long long rcp;
};
__device__ __forceinline__ ResDiv res_nodiv() {
    ResDiv D;
    D.o = 1; D.oinv = 1; D.p32 = D.Mch = D.mi = 0; D.rcp = 0;
    return D;
}
// row j of Toom-B: constants precomputed by the generator (toomgen emit_row_tables)
template <int B>
__device__ __forceinline__ ResDiv res_rowdiv(int j) {
    static_assert(RES_CH == 9, "tg_rowMch9 tables are for 9 positions per thread");
    ResDiv D;
    if constexpr (B == 3) {
        D.o = tg_rowO_T3[j]; D.oinv = tg_rowInv_T3[j]; D.p32 = tg_rowP32_T3[j]; D.Mch = tg_rowMch9_T3[j]; D.mi = tg_rowMi9_T3[j];
    } else {
        D.o = tg_rowO_T4[j]; D.oinv = tg_rowInv_T4[j]; D.p32 = tg_rowP32_T4[j]; D.Mch = tg_rowMch9_T4[j]; D.mi = tg_rowMi9_T4[j];
    }
    D.rcp = D.o > 1 ? ~0ull / D.o : 0ull;
    return D;
}

// One round of NT x CH positions: lin (this thread's positions r0 + tid*CH + q),
// state in sh.cin / sh.bin (uniform).  Writes the normalised (and, for o > 1,
// exactly divided) limbs through `put(q, limb)` and leaves the state at the
// round's end in sh.cin / sh.bin.  wt / wti: Mch^tid and mi^tid (o > 1).
template <class Put>
__device__ __forceinline__ void res_round(const long long (&lin)[RES_CH], const ResDiv& D, uint32_t wt, uint32_t wti,
                                          ResSmem& sh, Put put) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x, NW = NT >> 5;
    const uint32_t o = D.o;
    const LMod M{o, D.rcp};
    uint32_t x[RES_CH];
    long long c = 0;
#pragma unroll
    for (int q = 0; q < RES_CH; ++q) {
        const long long v = lin[q] + c;
        x[q] = (uint32_t)v;
        c = v >> 32;
    }
    LCMap A;
    {
        const unsigned long long L64 = (unsigned long long)x[0] | ((unsigned long long)x[1] << 32);
        bool tz = true, to = true;
#pragma unroll
        for (int q = 2; q < RES_CH; ++q) { tz &= (x[q] == 0u); to &= (x[q] == 0xFFFFFFFFu); }
        A.lo = (tz && L64 <= 0x8000000000000000ull) ? (long long)(0ull - L64) : LLONG_MIN;
        const unsigned long long comp = 0ull - L64;
        A.hi = (to && L64 != 0 && comp <= (unsigned long long)LLONG_MAX) ? (long long)comp : LLONG_MAX;
        A.cout[0] = c - 1;
        A.cout[1] = c;
        A.cout[2] = c + 1;
    }
    uint32_t s = 0;
    if (o > 1) {
        uint32_t r = 0;
#pragma unroll
        for (int q = RES_CH - 1; q >= 0; --q) r = lv_mod((unsigned long long)r * D.p32 + x[q], M);
        r = lv2_addmod(r, lv_mulmod(lv2_modc(c, M), D.Mch, M), o);
        s = lv_mulmod(r, wt, M);
    }
    LCMap inc = A;
    uint32_t sinc = s;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const LCMap prev = lc_shfl_up(inc, d);
        const uint32_t sp = __shfl_up_sync(0xffffffffu, sinc, d);
        if (lane >= d) {
            inc = lc_compose(prev, inc);
            if (o > 1) sinc = lv2_addmod(sinc, sp, o);
        }
    }
    const LCMap excl = lc_shfl_up(inc, 1);
    const uint32_t sexcl = __shfl_up_sync(0xffffffffu, sinc, 1);
    if (lane == 31) {
        sh.wmap[warp] = inc;
        sh.wres[warp] = sinc;
    }
    __syncthreads();
    long long cin = sh.cin;
    uint32_t Bt = 0;
    if (o > 1) Bt = lv2_addmod(lv2_modc(cin, M), sh.bin ? o - sh.bin : 0u, o);   // B at the round start
    uint32_t lam = 0;
    for (int w = 0; w < warp; ++w) {
        cin = lc_apply(sh.wmap[w], cin);
        if (o > 1) lam = lv2_addmod(lam, sh.wres[w], o);
    }
    if (lane > 0) {
        cin = lc_apply(excl, cin);
        if (o > 1) lam = lv2_addmod(lam, sexcl, o);
    }
    uint32_t beta = 0;
    if (o > 1) {
        const uint32_t bp = lv_mulmod(lv2_addmod(Bt, lam, o), wti, M);
        beta = lv2_addmod(lv2_modc(cin, M), bp ? o - bp : 0u, o);
    }
    c = cin;
#pragma unroll
    for (int q = 0; q < RES_CH; ++q) {
        const long long v = lin[q] + c;
        uint32_t xq = (uint32_t)v;
        c = v >> 32;
        if (o > 1) xq = tg_divexact_step(xq, beta, D.oinv, o);
        put(q, xq);
    }
    (void)NW;
    __syncthreads();   // every thread has read sh.cin / sh.bin / sh.wmap
    if (tid == NT - 1) {
        sh.cin = c;
        sh.bin = beta;
    }
    __syncthreads();
}

template <int B>
__device__ __forceinline__ long long res_evalc(int k, int j) {
    if constexpr (B == 3) return tg_evalc_T3[k][j];
    else return tg_evalc_T4[k][j];
}

// evaluation of one parent per CTA (blockIdx.y: operand 0 = u, 1 = v)
template <int B>
__global__ void __launch_bounds__(RES_MAXW * 32) k_res_eval(const uint32_t* __restrict__ srcU, const uint32_t* __restrict__ srcV,
                                                            uint32_t* __restrict__ dstU, uint32_t* __restrict__ dstV,
                                                            int count, int n, int b, int e, int sgn) {
    constexpr int NP = 2 * B - 1;
    extern __shared__ uint32_t rsm[];
    __shared__ ResSmem sh;
    const int tid = threadIdx.x, NT = blockDim.x;
    const long long c = blockIdx.x;
    const uint32_t* src = (blockIdx.y ? srcV : srcU) + c * (long long)n;
    uint32_t* dst = blockIdx.y ? dstV : dstU;
    uint32_t* P = rsm;   // [n]
    for (int i = tid; i < n; i += NT) P[i] = __ldg(src + i);
    __syncthreads();
    const int lentop = n - (B - 1) * b;
    const uint32_t fill = (sgn && (P[n - 1] >> 31)) ? 0xFFFFFFFFu : 0u;
    const int TL = NT * RES_CH;
    const ResDiv D = res_nodiv();
    for (int k = 0; k < NP; ++k) {
        long long cf[B];
#pragma unroll
        for (int j = 0; j < B; ++j) cf[j] = res_evalc<B>(k, j);
        uint32_t* out = dst + ((long long)k * count + c) * e;
        if (tid == 0) { sh.cin = 0; sh.bin = 0; }
        __syncthreads();
        for (int r0 = 0; r0 < e; r0 += TL) {
            const int p0 = r0 + tid * RES_CH;
            long long lin[RES_CH];
#pragma unroll
            for (int q = 0; q < RES_CH; ++q) {
                const int p = p0 + q;
                long long v = 0;
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    const int len = (j == B - 1) ? lentop : b;
                    const uint32_t x = p < len ? P[j * b + p] : (j == B - 1 ? fill : 0u);
                    v += cf[j] * (long long)x;
                }
                lin[q] = v;
            }
            res_round(lin, D, 1u, 1u, sh, [&](int q, uint32_t limb) {
                const int p = p0 + q;
                if (p < e) out[p] = limb;
            });
        }
    }
}

template <int B> __device__ __forceinline__ long long res_rowA(int j, int k) { return rowA<B>(j, k); }

// interpolation + recomposition of one parent per CTA
template <int B>
__global__ void __launch_bounds__(RES_MAXW * 32) k_res_interp(const uint32_t* __restrict__ Ysrc, uint32_t* __restrict__ dst,
                                                              long long dst_is, int count, int n, int b, int W2, int Lw) {
    constexpr int NP = 2 * B - 1;
    extern __shared__ uint32_t rsm[];
    __shared__ ResSmem sh;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NT = blockDim.x;
    const long long c = blockIdx.x;
    const int TL = NT * RES_CH;
    const int rounds = (Lw + 1 + TL - 1) / TL;
    uint32_t* Y = rsm;                                  // [NP][W2]
    uint32_t* R = Y + NP * W2;                          // [NP-2][Lw] interior coefficients
    uint32_t* Qb = R + (NP - 2) * Lw;                   // [rounds TL + 1] quotient limbs of a row
    for (int k = 0; k < NP; ++k) {
        const uint32_t* ys = Ysrc + ((long long)k * count + c) * W2;
        for (int i = tid; i < W2; i += NT) Y[k * W2 + i] = __ldg(ys + i);
    }
    __syncthreads();
    uint32_t fills[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) fills[k] = (Y[k * W2 + W2 - 1] >> 31) ? 0xFFFFFFFFu : 0u;
    // ---- interior coefficient rows
    for (int j = 1; j <= NP - 2; ++j) {
        long long A[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) A[k] = res_rowA<B>(j, k);
        const ResDiv D = res_rowdiv<B>(j);
        uint32_t wt = 1, wti = 1;
        if (D.o > 1) {
            const LMod M{D.o, D.rcp};
            wt = res_pow_tid(D.Mch, M, lane, warp);
            wti = res_pow_tid(D.mi, M, lane, warp);
        }
        if (tid == 0) { sh.cin = 0; sh.bin = 0; }
        __syncthreads();
        for (int rr = 0; rr < rounds; ++rr) {
            const int p0 = rr * TL + tid * RES_CH;
            long long lin[RES_CH];
#pragma unroll
            for (int q = 0; q < RES_CH; ++q) {
                const int p = p0 + q;
                long long v = 0;
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    if (A[k] == 0) continue;
                    const uint32_t x = p < W2 ? Y[k * W2 + p] : fills[k];
                    v += A[k] * (long long)x;
                }
                lin[q] = v;
            }
            res_round(lin, D, wt, wti, sh, [&](int q, uint32_t limb) { Qb[p0 + q] = limb; });
        }
        if (tg_check_on && tid == 0) {
            // dividend ended inside the window (rounds TL >= W2 limbs): carry and borrow
            // (csrc/check.cuh); the window holds y_k mod 2^(32 rounds TL)
            long long corr = 0;
#pragma unroll
            for (int k = 0; k < NP; ++k) corr += A[k] * (long long)(fills[k] & 1u);
            tg_check_end((uint64_t)(sh.cin - corr), sh.bin, D.o);
            tg_check_low(Qb[0], rowS<B>(j));
        }
        // the exact shift: w_j limb p = (Q[p], Q[p+1]) >> s
        const int s = rowS<B>(j);
        uint32_t* Rj = R + (j - 1) * Lw;
        for (int p = tid; p < Lw; p += NT) Rj[p] = __funnelshift_r(Qb[p], Qb[p + 1], s);
        __syncthreads();
    }
    // ---- recomposition w = sum_j w_j 2^(32 b j) (w_0 = y_0, w_2n = y_inf)
    auto rowlen = [&](int j) { return (j == 0 || j == NP - 1) ? W2 : Lw; };
    auto rowptr = [&](int j) -> const uint32_t* { return (j == 0 || j == NP - 1) ? Y + j * W2 : R + (j - 1) * Lw; };
    uint32_t rfill[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) rfill[j] = (rowptr(j)[rowlen(j) - 1] >> 31) ? 0xFFFFFFFFu : 0u;
    const int wout = 2 * n;
    uint32_t* out = dst + c * dst_is;
    if (tid == 0) { sh.cin = 0; sh.bin = 0; }
    __syncthreads();
    const ResDiv D1 = res_nodiv();
    for (int r0 = 0; r0 < wout; r0 += TL) {
        const int p0 = r0 + tid * RES_CH;
        long long lin[RES_CH];
#pragma unroll
        for (int q = 0; q < RES_CH; ++q) {
            const int P = p0 + q;
            unsigned long long v = 0;
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                const int i = P - j * b;
                if (i < 0) continue;
                v += (i < rowlen(j)) ? rowptr(j)[i] : rfill[j];
            }
            lin[q] = (long long)v;
        }
        res_round(lin, D1, 1u, 1u, sh, [&](int q, uint32_t limb) {
            const int P = p0 + q;
            if (P < wout) out[P] = limb;
        });
    }
}

inline size_t res_eval_smem(int n) { return (size_t)n * 4; }
inline size_t res_interp_smem(int B, int W2, int Lw, int nt) {
    const int NP = 2 * B - 1, TL = nt * RES_CH, rounds = (Lw + 1 + TL - 1) / TL;
    return 4 * ((size_t)NP * W2 + (size_t)(NP - 2) * Lw + (size_t)rounds * TL + 1);
}
// threads per CTA: enough warps for one round to cover the widest vector (<= 8 warps)
inline int res_threads(int W) {
    int w = (W + 32 * RES_CH - 1) / (32 * RES_CH);
    return 32 * std::max(1, std::min(RES_MAXW, w));
}

}  // namespace tg
