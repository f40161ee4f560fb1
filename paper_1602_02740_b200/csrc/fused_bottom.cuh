// Fused bottom Toom level (steps a2 + a3 + a4 + a5 of one
// recursion level whose children are base-case products), all in shared
// memory: no child operand, child product or coefficient ever touches HBM.
//
// CTA = G = 32 instances (one per lane) x NP = 2B-1 warps.
//   phase A  warp k  : evaluate U(x_k), V(x_k) for the 32 instances straight
//                      from the parent limbs (registers, E limbs each; table of
//                      homogeneous coefficients p^j q^(n-j)), multiply (register
//                      Comba, IMAD.WIDE.U32 carry chains), store the signed
//                      2E-limb product y_k in smem Y[k][t][lane]
//   phase B  warp j  : stream the coefficient w_j = (sum_k A_jk y_k) / D_j
//                      (the even-odd + Newton listing program composed into one
//                      row per coefficient; exact 2-adic division
//                      by the odd part of D_j, then the exact shift) into smem
//                      W[j][t][lane]
//   phase C  warp w  : recompose w = sum_j w_j 2^(32 b j) (Eq. 1.3) segment by
//                      segment (segment s = limbs [s b, s b + b)), each with a
//                      local carry chain; one lane per instance resolves the
//                      carries between segments; the segments then add their
//                      carry-in and write out (interleaved, or row-major at the
//                      top level through a coalesced smem copy)
// Phases A and B are table driven (one code path for every point / row) so the
// kernel stays small enough for the instruction cache.
#pragma once
#ifndef TG_FUSED_REG33
#define TG_FUSED_REG33 96   // measured: C4 bottom 970 -> 839 us, C3 504 -> 445 us
#endif
#ifndef TG_FUSED_REG18
#define TG_FUSED_REG18 64   // 64 registers: four CTAs per SM (measured 650 -> 596 us on C2)
#endif

namespace tg {

// parent operand accessor for the top level: row-major unsigned, block k limb t
struct FInTop {
    const uint32_t* row;
    int b, lentop, B;
    __device__ __forceinline__ uint32_t load(int k, int t) const {
        const int len = (k == B - 1) ? lentop : b;
        return (t < len) ? __ldg(row + k * b + t) : 0u;
    }
};

// parent operand staged in smem: block k limb t at P[(k*b + t)*33]
struct SmemParent {
    const uint32_t* P;
    int b, lentop, B;
    uint32_t fill;   // sign fill of the top block (0 at the top level)
    __device__ __forceinline__ uint32_t load(int k, int t) const {
        const int len = (k == B - 1) ? lentop : b;
        if (t < len) return P[(k * b + t) * 33];
        return (k == B - 1) ? fill : 0u;
    }
};

template <int B>
__device__ __forceinline__ long long evalc(int k, int j) {
    if constexpr (B == 3) return tg_evalc_T3[k][j];
    else return tg_evalc_T4[k][j];
}
template <int B>
__device__ __forceinline__ long long rowA(int j, int k) {
    if constexpr (B == 3) return tg_rowA_T3[j][k];
    else return tg_rowA_T4[j][k];
}
template <int B> __device__ __forceinline__ uint32_t rowO(int j) { if constexpr (B == 3) return tg_rowO_T3[j]; else return tg_rowO_T4[j]; }
template <int B> __device__ __forceinline__ uint32_t rowInv(int j) { if constexpr (B == 3) return tg_rowInv_T3[j]; else return tg_rowInv_T4[j]; }
template <int B> __device__ __forceinline__ int rowS(int j) { if constexpr (B == 3) return tg_rowS_T3[j]; else return tg_rowS_T4[j]; }

// evaluation of point k: r = sum_j c[k][j] * block_j, E limbs, LSB first with a
// signed 64-bit carry (two's-complement result)
template <int B, int E, class In>
__device__ __forceinline__ void eval_point(int k, const In& in, uint32_t (&r)[E]) {
    uint64_t c[B];
#pragma unroll
    for (int j = 0; j < B; ++j) c[j] = (uint64_t)evalc<B>(k, j);
    uint64_t acc = 0;
#pragma unroll
    for (int t = 0; t < E; ++t) {
        uint64_t lin = acc;
#pragma unroll
        for (int j = 0; j < B; ++j) lin += c[j] * (uint64_t)in.load(j, t);
        r[t] = (uint32_t)lin;
        acc = (uint64_t)((int64_t)lin >> 32);
    }
}

// interpolation row j: w_j = (sum_k A[j][k] y_k) / (o_j 2^s_j); y_k read from
// smem Yl[(k*w2 + t)*32] (sign-extended past w2), w_j written to dst[t*32] for
// t < Lw.  The shift is applied one limb late (s = 0 is a plain delay).
template <int B>
__device__ __forceinline__ void interp_row(int j, const uint32_t* __restrict__ Yl, int w2, uint32_t* __restrict__ dst,
                                           int Lw) {
    constexpr int NP = 2 * B - 1;
    uint64_t A[NP];
    uint32_t fill[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        A[k] = (uint64_t)rowA<B>(j, k);
        fill[k] = (Yl[(k * w2 + w2 - 1) * 32] >> 31) ? 0xFFFFFFFFu : 0u;
    }
    const uint32_t o = rowO<B>(j), oinv = rowInv<B>(j);
    const int sh = rowS<B>(j);
    uint64_t acc = 0;
    uint32_t bor = 0, qp = 0;
#pragma unroll 1
    for (int t = 0; t <= Lw; ++t) {
        uint64_t lin = acc;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            const uint32_t y = (t < w2) ? Yl[(k * w2 + t) * 32] : fill[k];
            lin += A[k] * (uint64_t)y;
        }
        acc = (uint64_t)((int64_t)lin >> 32);
        const uint32_t q = tg_divexact_step((uint32_t)lin, bor, oinv, o);
        if (t > 0) dst[(t - 1) * 32] = __funnelshift_r(qp, q, sh);
        qp = q;
    }
}

template <int B, int E>
__device__ __forceinline__ void eval_point_regs(int k, const uint32_t* PU, const uint32_t* PV, uint32_t (&a)[E],
                                                uint32_t (&b)[E]) {
    if constexpr (B == 3) {
        switch (k) {
            case 0: tg_evalreg_T3_0<E>(PU, PV, a, b); break;
            case 1: tg_evalreg_T3_1<E>(PU, PV, a, b); break;
            case 2: tg_evalreg_T3_2<E>(PU, PV, a, b); break;
            case 3: tg_evalreg_T3_3<E>(PU, PV, a, b); break;
            default: tg_evalreg_T3_4<E>(PU, PV, a, b); break;
        }
    } else {
        switch (k) {
            case 0: tg_evalreg_T4_0<E>(PU, PV, a, b); break;
            case 1: tg_evalreg_T4_1<E>(PU, PV, a, b); break;
            case 2: tg_evalreg_T4_2<E>(PU, PV, a, b); break;
            case 3: tg_evalreg_T4_3<E>(PU, PV, a, b); break;
            case 4: tg_evalreg_T4_4<E>(PU, PV, a, b); break;
            case 5: tg_evalreg_T4_5<E>(PU, PV, a, b); break;
            default: tg_evalreg_T4_6<E>(PU, PV, a, b); break;
        }
    }
}

template <int B, int E>
__device__ __forceinline__ void eval_point_rows(int k, const uint32_t* PU, const uint32_t* PV, uint32_t* dU, uint32_t* dV) {
    if constexpr (B == 3) {
        switch (k) {
            case 0: tg_evalrow_T3_0<E>(PU, PV, dU, dV); break;
            case 1: tg_evalrow_T3_1<E>(PU, PV, dU, dV); break;
            case 2: tg_evalrow_T3_2<E>(PU, PV, dU, dV); break;
            case 3: tg_evalrow_T3_3<E>(PU, PV, dU, dV); break;
            default: tg_evalrow_T3_4<E>(PU, PV, dU, dV); break;
        }
    } else {
        switch (k) {
            case 0: tg_evalrow_T4_0<E>(PU, PV, dU, dV); break;
            case 1: tg_evalrow_T4_1<E>(PU, PV, dU, dV); break;
            case 2: tg_evalrow_T4_2<E>(PU, PV, dU, dV); break;
            case 3: tg_evalrow_T4_3<E>(PU, PV, dU, dV); break;
            case 4: tg_evalrow_T4_4<E>(PU, PV, dU, dV); break;
            case 5: tg_evalrow_T4_5<E>(PU, PV, dU, dV); break;
            default: tg_evalrow_T4_6<E>(PU, PV, dU, dV); break;
        }
    }
}

// two's-complement product of two E-limb two's-complement operands, 2E limbs
// to dst[t*32]: the unsigned product A*B (Comba, IMAD.WIDE.U32 carry chains)
// minus 2^(32E) * (sa*B + sb*A) (mod 2^(64E)), applied to the top E limbs.
template <int E>
__device__ __forceinline__ void mul_twos_to_smem(const uint32_t (&a)[E], const uint32_t (&b)[E], uint32_t* dst) {
    const uint32_t ma = 0u - (a[E - 1] >> 31), mb = 0u - (b[E - 1] >> 31);
    uint32_t c0 = 0, c1 = 0, c2 = 0;
    // low half: plain columns
#pragma unroll
    for (int k = 0; k < E; ++k) {
#pragma unroll
        for (int i = 0; i <= k; ++i) TG_MADD(c0, c1, c2, a[i], b[k - i]);
        dst[k * 32] = c0;
        c0 = c1; c1 = c2; c2 = 0;
    }
    // high half: columns minus the correction, borrow chain in `br`
    uint32_t br = 0;
#pragma unroll
    for (int k = E; k < 2 * E; ++k) {
        if (k < 2 * E - 1) {
#pragma unroll
            for (int i = k - E + 1; i <= E - 1; ++i) TG_MADD(c0, c1, c2, a[i], b[k - i]);
        }
        const uint64_t sub = (uint64_t)(b[k - E] & ma) + (a[k - E] & mb) + br;
        const uint64_t x = (uint64_t)c0 - (uint32_t)sub;
        dst[k * 32] = (uint32_t)x;
        br = (uint32_t)(sub >> 32) + (uint32_t)((x >> 32) & 1u);
        c0 = c1; c1 = c2; c2 = 0;
    }
}

// squaring specialisation: a^2 = |a|^2 of an E-limb two's-
// complement value, 2E limbs to dst[t*32]: the cross products
// sum_{i<j} a_i a_j 2^(32(i+j)) by product scanning (E(E-1)/2 limb-products
// instead of E^2), then doubled and the diagonal squares a_i^2 2^(64 i) added
// in one carry pass over the limbs.
template <int E>
__device__ __forceinline__ void sqr_twos_to_smem(uint32_t (&a)[E], uint32_t* dst) {
    {
        const uint32_t sa = a[E - 1] >> 31, m = 0u - sa;
        uint32_t cy = sa;
#pragma unroll
        for (int i = 0; i < E; ++i) { const uint32_t x = (a[i] ^ m) + cy; cy = (x < cy) ? 1u : 0u; a[i] = x; }
    }
    uint32_t c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
    for (int k = 1; k < 2 * E - 2; ++k) {
#pragma unroll
        for (int i = (k < E ? 0 : k - E + 1); 2 * i < k; ++i) TG_MADD(c0, c1, c2, a[i], a[k - i]);
        dst[k * 32] = c0;
        c0 = c1; c1 = c2; c2 = 0;
    }
    dst[(2 * E - 2) * 32] = c0;
    dst[(2 * E - 1) * 32] = c1;
    // w = 2 C + sum_i a_i^2 2^(64 i): limb k gets (C_k << 1 | C_{k-1} >> 31) and
    // the low (k even) or high (k odd) word of a_{k/2}^2
    uint64_t acc = 0;
    uint32_t prev = 0;   // C_{k-1}
#pragma unroll
    for (int k = 0; k < 2 * E; ++k) {
        const uint32_t ck = k >= 1 ? dst[k * 32] : 0u;
        const uint32_t dbl = (ck << 1) | (prev >> 31);
        prev = ck;
        const uint64_t sq = (uint64_t)a[k >> 1] * a[k >> 1];
        acc += (uint64_t)dbl + ((k & 1) ? (uint32_t)(sq >> 32) : (uint32_t)sq);
        dst[k * 32] = (uint32_t)acc;
        acc >>= 32;
    }
}

// |a| * |b| with the product sign applied, 2E limbs streamed to dst[t*32]
template <int E>
__device__ __forceinline__ void mul_signed_to_smem(uint32_t (&a)[E], uint32_t (&b)[E], uint32_t* dst) {
    uint32_t sa = a[E - 1] >> 31, sb = b[E - 1] >> 31;
    {
        const uint32_t m = 0u - sa;
        uint32_t cy = sa;
#pragma unroll
        for (int i = 0; i < E; ++i) { const uint32_t x = (a[i] ^ m) + cy; cy = (x < cy) ? 1u : 0u; a[i] = x; }
    }
    {
        const uint32_t m = 0u - sb;
        uint32_t cy = sb;
#pragma unroll
        for (int i = 0; i < E; ++i) { const uint32_t x = (b[i] ^ m) + cy; cy = (x < cy) ? 1u : 0u; b[i] = x; }
    }
    const uint32_t neg = sa ^ sb, mask = 0u - neg;
    uint32_t ncarry = neg, c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
    for (int k = 0; k < 2 * E - 1; ++k) {
#pragma unroll
        for (int i = (k < E ? 0 : k - E + 1); i <= (k < E ? k : E - 1); ++i) TG_MADD(c0, c1, c2, a[i], b[k - i]);
        const uint32_t x = (c0 ^ mask) + ncarry;
        ncarry = (x < ncarry) ? 1u : 0u;
        dst[k * 32] = x;
        c0 = c1; c1 = c2; c2 = 0;
    }
    dst[(2 * E - 1) * 32] = (c0 ^ mask) + ncarry;
}

// shared memory bytes for a launch (Y | W | per-segment carries)
// shared memory words of the W region (coefficient rows; the parents are
// staged there first).  MODE 0 keeps only the interior rows 1..2B-3 (w_0 and
// w_2n are read from the products) and two carry arrays, so that four CTAs
// fit per SM.
__host__ __device__ inline size_t fused_wreg(int B, int E, int Lw, int mode) {
    const int NP = 2 * B - 1;
    size_t wreg = (size_t)(mode == 0 ? NP - 2 : NP) * Lw * 32;
    if ((size_t)2 * B * E * 33 > wreg) wreg = (size_t)2 * B * E * 33;   // parents staged in the W region
    return wreg;
}
__host__ __device__ inline size_t fused_smem_bytes(int B, int E, int Lw, int nseg, int n, int mode) {
    const int NP = 2 * B - 1;
    return (size_t)4 * ((size_t)NP * 2 * E * 32 + fused_wreg(B, E, Lw, mode) + (mode == 0 ? 2 : 4) * 32 * (size_t)nseg);
}

// diagnostic phase mask (bench/debug only; all phases by default): bit 0
// products, bit 1 rows, bit 2 recomposition.  Results are wrong when a phase
// is masked; used to measure the phases' share of the kernel time.
__device__ int tg_fused_phase_mask = 7;

// MODE: 0 = parents interleaved [n][count], signed (a lower level of a batch);
//       1 = parents row-major [count][n], unsigned (the top level);
//       2 = parents row-major [count][n], signed (below a long-vector level);
//       3 = parents interleaved, signed, products row-major (below a top level
//           whose interpolation runs one warp per product).
// Output products: interleaved [2n][count] for MODE 0, row-major [count][2n]
// otherwise.
// N_, BB_ != 0 fix n and b (hence Lw = 2b+1, wout = 2n, nseg) at compile time
// (the C2 shape): shared-memory offsets and trip counts become immediates.
template <int B, int E, int MODE, int N_ = 0, int BB_ = 0, bool SQ = false>
__global__ void __maxnreg__(E <= 18 ? TG_FUSED_REG18 : TG_FUSED_REG33) k_fused_bottom(
    const uint32_t* __restrict__ srcU, const uint32_t* __restrict__ srcV, uint32_t* __restrict__ out,
    size_t count, int n_, int b_, int Lw_, int wout_, int nseg_) {
    constexpr bool ST = N_ != 0 && BB_ != 0;
    const int n = ST ? N_ : n_;
    const int b = ST ? BB_ : b_;
    const int Lw = ST ? 2 * BB_ + 1 : Lw_;
    const int wout = ST ? 2 * N_ : wout_;
    const int nseg = ST ? (2 * N_ + BB_ - 1) / BB_ : nseg_;
    constexpr int NP = 2 * B - 1;
    constexpr int G = 32;
    extern __shared__ uint32_t sm[];
    uint32_t* Y = sm;                          // [NP][2E][G], later OUT [wout][G]
    uint32_t* Wb = Y + NP * 2 * E * G;         // [NP][Lw][G]  (MODE 0: [NP-2][Lw][G])
    const int wreg = (int)fused_wreg(B, E, Lw, MODE);
    uint32_t* CO = Wb + wreg;                  // [nseg][G] segment carry-out
    uint32_t* L0 = CO + nseg * G;              // [nseg][G] limb 0 of the segment
    uint32_t* ON = L0 + nseg * G;              // [nseg][G] limbs 1.. all ones
    uint32_t* CI = ON + nseg * G;              // [nseg][G] resolved carry-in
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const size_t c = (size_t)blockIdx.x * G + lane;
    const bool valid = c < count;
    const int lentop = n - (B - 1) * b;

    // ---- phase A0: stage the 32 parents' operand blocks in smem (W region,
    // unused until phase B), padded to E limbs per block (zero fill, sign fill
    // for the top block below the top level): P[op][j][t][33]
    constexpr int PP = 33;                     // padded pitch (conflict-free transpose)
    uint32_t* Pu = Wb;
    uint32_t* Pv = Wb + B * E * PP;
    {
        const size_t c0 = (size_t)blockIdx.x * G;
        const int nin = (int)min((size_t)G, count - c0);
        // rows t of block j: source limb j*b + t when t < len_j; all loads of
        // a warp are issued before its stores (compile-time trip count)
        uint32_t fu = 0, fv = 0;
        if ((MODE == 0 || MODE == 3) && lane < nin) {
            fu = (__ldg(srcU + (size_t)(n - 1) * count + c0 + lane) >> 31) ? 0xFFFFFFFFu : 0u;
            fv = (__ldg(srcV + (size_t)(n - 1) * count + c0 + lane) >> 31) ? 0xFFFFFFFFu : 0u;
        }
        if (MODE == 2 && lane < nin) {
            fu = (__ldg(srcU + (c0 + lane) * (size_t)n + n - 1) >> 31) ? 0xFFFFFFFFu : 0u;
            fv = (__ldg(srcV + (c0 + lane) * (size_t)n + n - 1) >> 31) ? 0xFFFFFFFFu : 0u;
        }
        constexpr int ROWS = B * E, ITER = (ROWS + NP - 1) / NP;
        if constexpr (ST && (MODE == 0 || MODE == 3) && B * E - N_ <= NP && E > BB_) {
            // compile-time shape: source limb row l (coalesced across the 32
            // parents) is block j = min(l / b, B - 1), limb l - j b, smem row
            // l + j (E - b); the B E - n pad rows (zero, or the sign fill of
            // the top block) take one warp each
            constexpr int IT = (N_ + NP - 1) / NP, LT = N_ - (B - 1) * BB_, NPAD = B * E - N_;
            const size_t stp = (size_t)NP * count;
            const uint32_t* pu = srcU + (size_t)warp * count + c0 + lane;
            const uint32_t* pv = srcV + (size_t)warp * count + c0 + lane;
            uint32_t yu[IT], yv[IT];
#pragma unroll
            for (int q = 0; q < IT; ++q) {
                const int l = warp + NP * q;
                yu[q] = yv[q] = 0u;
                if (l < N_ && lane < nin) {
                    yu[q] = __ldg(pu);
                    yv[q] = __ldg(pv);
                }
                pu += stp;
                pv += stp;
            }
#pragma unroll
            for (int q = 0; q < IT; ++q) {
                const int l = warp + NP * q;
                if (l < N_) {
                    const int j = min(l / BB_, B - 1);
                    const int r = l + j * (E - BB_);
                    Pu[r * PP + lane] = yu[q];
                    Pv[r * PP + lane] = yv[q];
                }
            }
            if (warp < NPAD) {
                // pad row `warp`: rows j E + [b, E) of blocks j < B - 1 (zero),
                // then (B - 1) E + [lentop, E) of the top block (fill)
                constexpr int ZP = (B - 1) * (E - BB_);
                const int r = warp < ZP ? (warp / (E - BB_)) * E + BB_ + warp % (E - BB_) : (B - 1) * E + LT + (warp - ZP);
                Pu[r * PP + lane] = warp < ZP ? 0u : fu;
                Pv[r * PP + lane] = warp < ZP ? 0u : fv;
            }
        } else {
        uint32_t xu[ITER], xv[ITER];
        if constexpr (MODE == 0 || MODE == 3) {
            // interleaved parents: row r = warp + q NP is block j limb t; both
            // advance incrementally and the source pointers by whole limb rows
            int j = warp / E, t = warp - (warp / E) * E;
            const uint32_t* pu = srcU + (size_t)(j * b + t) * count + c0 + lane;
            const uint32_t* pv = srcV + (size_t)(j * b + t) * count + c0 + lane;
#pragma unroll
            for (int q = 0; q < ITER; ++q) {
                const int r = warp + q * NP;
                const int len = (j == B - 1) ? lentop : b;
                xu[q] = 0;
                xv[q] = 0;
                if (r < ROWS && lane < nin) {
                    if (t < len) {
                        xu[q] = __ldg(pu);
                        xv[q] = __ldg(pv);
                    } else if (j == B - 1) {
                        xu[q] = fu;
                        xv[q] = fv;
                    }
                }
                if (q + 1 < ITER) {
                    int dl = NP;
                    t += NP;
                    while (t >= E) { t -= E; ++j; dl += b - E; }
                    pu += (long long)dl * (long long)count;
                    pv += (long long)dl * (long long)count;
                }
            }
        } else {
#pragma unroll
        for (int q = 0; q < ITER; ++q) {
            const int r = warp + q * NP;
            const int j = r / E, t = r - j * E;
            const int len = (j == B - 1) ? lentop : b;
            const int limb = j * b + t;
            xu[q] = 0;
            xv[q] = 0;
            if (r < ROWS && lane < nin) {
                if (t < len) {
                    if (MODE == 1 || MODE == 2) {
                        xu[q] = __ldg(srcU + (c0 + lane) * (size_t)n + limb);
                        xv[q] = __ldg(srcV + (c0 + lane) * (size_t)n + limb);
                    } else {
                        xu[q] = __ldg(srcU + (size_t)limb * count + c0 + lane);
                        xv[q] = __ldg(srcV + (size_t)limb * count + c0 + lane);
                    }
                } else if (j == B - 1) {
                    xu[q] = fu;
                    xv[q] = fv;
                }
            }
        }
        }
#pragma unroll
        for (int q = 0; q < ITER; ++q) {
            const int r = warp + q * NP;
            if (r < ROWS) {
                Pu[r * PP + lane] = xu[q];
                Pv[r * PP + lane] = xv[q];
            }
        }
        }
    }
    __syncthreads();

    const int pmask = tg_fused_phase_mask;
    // ---- phase A: evaluate point `warp` of both operands (from smem) into
    // the warp's own Y[k] slot, load to registers, multiply into the same slot
    if (valid) {
        // (the rolled smem evaluation keeps the kernel small enough for the
        // instruction cache; a fully unrolled register version measured slower)
        uint32_t* slot = Y + (warp * 2 * E) * G + lane;
        eval_point_rows<B, E>(warp, Pu + lane, Pv + lane, slot, slot + E * G);
        uint32_t a[E], bb[E];
#pragma unroll
        for (int t = 0; t < E; ++t) { a[t] = slot[t * G]; bb[t] = slot[(E + t) * G]; }
        if (pmask & 1) {
            if constexpr (SQ) sqr_twos_to_smem<E>(a, slot);   // V = U: the square
            else mul_twos_to_smem<E>(a, bb, slot);
        }
        // fault injection (tests): one flipped bit of y_1 of the
        // CTA's first instance makes the rows' exact divisions inexact
        if (tg_fault == 1 && blockIdx.x == 0 && lane == 0 && warp == 1) slot[3 * G] ^= 1u;
    }
    __syncthreads();

    // ---- phase B: coefficient w_warp (w_0 = y_0 and w_2n = y_inf are copies)
    if (valid && (pmask & 2)) {
        const uint32_t* Yl = Y + lane;
        uint32_t* dst = Wb + ((MODE == 0 ? warp - 1 : warp) * Lw) * G + lane;
        if (warp == 0 || warp == NP - 1) {
            // MODE 0 reads w_0 = y_0 and w_2n = y_inf straight from the products;
            // warp 0 (idle otherwise) writes recomposition segment 0 now: its
            // limbs are w_0[0..b) = y_0[0..b) alone, with carry-out 0
            if constexpr (MODE == 0) {
                if (warp == 0) {
                    const uint32_t* src = Yl;
                    const int len = min(b, wout);
                    for (int r = 0; r < len; ++r) out[(size_t)r * count + c] = src[r * G];
                    CO[lane] = 0u;
                    CO[nseg * G + lane] = 0u;
                }
            } else {
                const uint32_t* src = Yl + (warp * 2 * E) * G;
                for (int t = 0; t < Lw; ++t) dst[t * G] = src[t * G];
            }
        } else if constexpr (B == 3) {
            // (the destination row is recomputed per case so that, with a
            // compile-time shape, its offset from Yl is an immediate)
#define TG_DST(J) (Wb + ((MODE == 0 ? (J) - 1 : (J)) * Lw) * G + lane)
            switch (warp) {
                case 1: tg_row_T3_1<2 * E>(Yl, TG_DST(1), Lw); break;
                case 2: tg_row_T3_2<2 * E>(Yl, TG_DST(2), Lw); break;
                default: tg_row_T3_3<2 * E>(Yl, TG_DST(3), Lw); break;
            }
        } else {
            switch (warp) {
                case 1: tg_row_T4_1<2 * E>(Yl, TG_DST(1), Lw); break;
                case 2: tg_row_T4_2<2 * E>(Yl, TG_DST(2), Lw); break;
                case 3: tg_row_T4_3<2 * E>(Yl, TG_DST(3), Lw); break;
                case 4: tg_row_T4_4<2 * E>(Yl, TG_DST(4), Lw); break;
                default: tg_row_T4_5<2 * E>(Yl, TG_DST(5), Lw); break;
            }
#undef TG_DST
        }
    }
    __syncthreads();

    if (!(pmask & 4)) return;
    if constexpr (MODE == 0) {
        // ---- phase C (interleaved output): recompose w = sum_j w_j 2^(32 b j)
        // segment by segment; the products stay intact (w_0, w_2n are read
        // from them), so a carry-out pass, the carry resolution between
        // segments and a final pass that writes straight to global memory.
        auto rowp = [&](int j) -> const uint32_t* {
            return (j == 0 || j == NP - 1) ? Y + (j * 2 * E) * G + lane : Wb + ((j - 1) * Lw) * G + lane;
        };
        auto fillj = [&](int j) -> uint32_t { return rowp(j)[(Lw - 1) * G] >> 31; };
        // segment s: limb r = w_s[r] + w_{s-1}[b + r] (+ w_{s-2}[2b] at r = 0)
        // + the sign fills of the rows that have ended
        auto seg = [&](int s, uint64_t cin, bool write, uint32_t* l0o, uint32_t* oneso) -> uint64_t {
            uint32_t lowfills = 0, fillC = 0;
            for (int j = 0; j <= s - 2 && j < NP; ++j) {
                const uint32_t f = fillj(j);
                if (j == s - 2) fillC = f;
                else lowfills += f;
            }
            const bool hasA = s < NP, hasB = s >= 1 && s - 1 < NP, hasC = s >= 2 && s - 2 < NP;
            const uint32_t* pA = hasA ? rowp(s) : nullptr;
            const uint32_t* pB = hasB ? rowp(s - 1) + b * G : nullptr;
            const int P0 = s * b;
            const int len = min(b, wout - P0);
            uint64_t x = cin + (uint64_t)lowfills * 0xFFFFFFFFull;
            if (hasA) x += pA[0];
            if (hasB) x += pB[0];
            if (hasC) x += rowp(s - 2)[(2 * b) * G];
            uint32_t lo = (uint32_t)x;
            if (l0o) *l0o = lo;
            if (write) out[(size_t)P0 * count + c] = lo;
            uint64_t carry = x >> 32;
            const uint64_t cc = (uint64_t)(lowfills + fillC) * 0xFFFFFFFFull;
            uint32_t ones = 0xFFFFFFFFu;
            if (hasA && hasB) {
                for (int r = 1; r < len; ++r) {
                    const uint64_t y = carry + cc + pA[r * G] + pB[r * G];
                    lo = (uint32_t)y;
                    if (write) out[(size_t)(P0 + r) * count + c] = lo;
                    ones &= lo;
                    carry = y >> 32;
                }
            } else {
                for (int r = 1; r < len; ++r) {
                    uint64_t y = carry + cc;
                    if (hasA) y += pA[r * G];
                    if (hasB) y += pB[r * G];
                    lo = (uint32_t)y;
                    if (write) out[(size_t)(P0 + r) * count + c] = lo;
                    ones &= lo;
                    carry = y >> 32;
                }
            }
            if (oneso) *oneso = ones;
            return carry;
        };
        // CO[s] = carry-out | (limbs 1.. all ones) << 31, later the resolved carry-in
        uint32_t* L0c = CO + nseg * G;
        // one pass: every segment is written with carry-in 0; the resolved
        // carry-ins are added afterwards (they rarely ripple past limb 0)
        if (valid) {
            for (int s = warp + 1; s < nseg; s += NP) {   // segment 0 was written in phase B
                uint32_t l0, ones;
                const uint64_t cout = seg(s, 0, true, &l0, &ones);
                CO[s * G + lane] = (uint32_t)cout | ((ones == 0xFFFFFFFFu) ? 0x80000000u : 0u);
                L0c[s * G + lane] = l0;
            }
        }
        __syncthreads();
        if (valid && warp == 0) {
            uint32_t cin = 0;
            for (int s = 0; s < nseg; ++s) {
                const uint32_t co = CO[s * G + lane];
                uint32_t cout = co & 0x7FFFFFFFu;
                if (cin) {
                    const uint32_t l0 = L0c[s * G + lane];
                    if (l0 + cin < l0 && (co >> 31)) cout += 1;
                }
                CO[s * G + lane] = cin;
                cin = cout;
            }
        }
        __syncthreads();
        if (valid) {
            for (int s = warp + 1; s < nseg; s += NP) {
                uint32_t cin = CO[s * G + lane];
                const int P0 = s * b;
                const int len = min(b, wout - P0);
                for (int r = 0; r < len && cin; ++r) {
                    uint32_t* po = out + (size_t)(P0 + r) * count + c;
                    const uint32_t x = *po;
                    const uint32_t y = x + cin;
                    *po = y;
                    cin = (y < x) ? 1u : 0u;
                }
            }
        }
        return;
    }
    // ---- phase C1: segment sums with local carries (OUT aliases Y)
    uint32_t* OUT = Y;
    if (valid) {
        for (int s = warp; s < nseg; s += NP) {
            uint32_t lowfills = 0, fillC = 0;
            for (int j = 0; j <= s - 2 && j < NP; ++j) {
                const uint32_t f = Wb[(j * Lw + Lw - 1) * G + lane] >> 31;
                if (j == s - 2) fillC = f;
                else lowfills += f;
            }
            const bool hasA = s < NP, hasB = s >= 1 && s - 1 < NP, hasC = s >= 2 && s - 2 < NP;
            const uint32_t* pA = Wb + ((hasA ? s : 0) * Lw) * G + lane;
            const uint32_t* pB = Wb + ((hasB ? s - 1 : 0) * Lw + b) * G + lane;
            const int P0 = s * b;
            const int len = min(b, wout - P0);
            uint64_t acc = (uint64_t)lowfills * 0xFFFFFFFFull;
            if (hasA) acc += pA[0];
            if (hasB) acc += pB[0];
            if (hasC) acc += Wb[((s - 2) * Lw + 2 * b) * G + lane];
            uint32_t limb0 = (uint32_t)acc;
            OUT[P0 * G + lane] = limb0;
            uint64_t carry = acc >> 32;
            const uint64_t cc = (uint64_t)(lowfills + fillC) * 0xFFFFFFFFull;
            uint32_t ones = 0xFFFFFFFFu;
            for (int r = 1; r < len; ++r) {
                uint64_t x = carry + cc;
                if (hasA) x += pA[r * G];
                if (hasB) x += pB[r * G];
                const uint32_t lo = (uint32_t)x;
                OUT[(P0 + r) * G + lane] = lo;
                ones &= lo;
                carry = x >> 32;
            }
            CO[s * G + lane] = (uint32_t)carry;
            L0[s * G + lane] = limb0;
            ON[s * G + lane] = (ones == 0xFFFFFFFFu) ? 1u : 0u;
        }
    }
    __syncthreads();
    // ---- phase C2: resolve the carries between segments (one lane per instance)
    if (valid && warp == 0) {
        uint32_t cin = 0;
        for (int s = 0; s < nseg; ++s) {
            CI[s * G + lane] = cin;
            uint32_t cout = CO[s * G + lane];
            if (cin) {
                const uint32_t l0 = L0[s * G + lane];
                if (l0 + cin < l0 && ON[s * G + lane]) cout += 1;
            }
            cin = cout;
        }
    }
    __syncthreads();
    // ---- phase C3: apply carry-in, write out
    if (valid) {
        for (int s = warp; s < nseg; s += NP) {
            uint32_t cin = CI[s * G + lane];
            const int P0 = s * b;
            const int len = min(b, wout - P0);
            for (int r = 0; r < len && cin; ++r) {
                const uint32_t x = OUT[(P0 + r) * G + lane];
                const uint32_t y = x + cin;
                cin = (y < x) ? 1u : 0u;
                OUT[(P0 + r) * G + lane] = y;
            }
            if (MODE == 0)
                for (int r = 0; r < len; ++r) out[(size_t)(P0 + r) * count + c] = OUT[(P0 + r) * G + lane];
        }
    }
    if (MODE != 0) {
        __syncthreads();
        // coalesced row-major copy: w[c0 + i][P]
        const size_t c0 = (size_t)blockIdx.x * G;
        const int rows = (int)min((size_t)G, count - c0);
        for (int idx = threadIdx.x; idx < rows * wout; idx += blockDim.x) {
            const int i = idx / wout, P = idx - i * wout;
            out[(c0 + i) * (size_t)wout + P] = OUT[P * G + i];
        }
    }
}

}  // namespace tg
