// Top-level interpolation + recomposition of the C2 shape (Toom-4, n = 256,
// b = 64; 130-limb child products, interleaved) as ONE division over the
// common denominator (steps a4 + a5; reading 18):
//     D w = X = sum_j 2^(32 b j) sum_k A'_jk y_k        (A' = tg_combA_T4)
// with D = 360, or D = 360 * 360 when the children come from the deferred
// bottom (csrc/fused_dc.cuh: y_k = 360 y'_k).  The matrix form
// has no division, so limb P of X,
//     X[P] = sum_j sum_k A'_jk y_k[P - 64 j]     (|X[P]| < 2^45),
// is elementwise in P; the one exact division by D = 2^s o (2-adic by o, ref
// [4], then a shift) is split into segments of positions whose
// borrow-in comes from the closed form
//     beta_p = (c_p - 2^(-32 p) sum_{i<p} X_i 2^(32 i)) mod o
// (c_p the carry into p), so every warp works in every phase:
//   0  stage the 7 products of G = 28 parents (cp.async, [k][t][G])
//   1  class r = P mod 64 (warp w: r = w, w + 7, ...): the columns t = r,
//      r + 64 (, r + 128 / the sign column 130) give X[r + 64 m], m = 0..8,
//      written over the class's own columns (lo words, packed 16-bit highs)
//   2  segment s (warp s of 14): carries with carry-in 0 -> limbs z, the carry-out
//      and the residue of the segment's X mod o
//   3  warp s: its carry-in (the previous segment's carry-out) and borrow-in
//      (closed form over the earlier segments' residues); a carry that wraps
//      a limb 0 (~2^-17) sends the product through warp 0's serial chain
//   4  segment s: the 2-adic division chain from its borrow-in
//   5  all warps: w = q >> s to the row-major output (16-byte stores)
#pragma once

namespace tg {

namespace cls {
constexpr int NP = 7, BB = 64, YW = 130, G = 28, WOUT = 512, NPOS = 513;
constexpr int NW = 14, NSEG = NW;   // warps per CTA (two CTAs per SM by shared memory), one segment each
__host__ __device__ constexpr int seg0(int s) { return 36 * s + (s > 5 ? s - 5 : 0); }
static_assert(seg0(NSEG) == NPOS, "segments cover the 513 quotient limbs");
__host__ __device__ constexpr uint32_t modpow32(uint32_t o, long long e) {   // 2^(32 e) mod o, e >= 0
    uint64_t r = 1 % o, b = (uint64_t)(((unsigned __int128)1 << 32) % o);
    while (e) { if (e & 1) r = r * b % o; b = b * b % o; e >>= 1; }
    return (uint32_t)r;
}
__host__ __device__ constexpr uint32_t invmod(uint32_t a, uint32_t o) {   // a^-1 mod o (gcd = 1)
    long long t = 0, nt = 1, r = o, nr = a % o;
    while (nr) { const long long q = r / nr, x = t - q * nt; t = nt; nt = x; const long long y = r - q * nr; r = nr; nr = y; }
    return (uint32_t)(t < 0 ? t + o : t);
}
__host__ __device__ constexpr uint32_t inv32(uint32_t o) {
    uint32_t x = o;
    for (int i = 0; i < 5; ++i) x *= 2u - o * x;
    return x;
}
template <bool DEF> struct Den {
    static constexpr uint32_t o = DEF ? 2025u : 45u;   // odd part of 360 (or 360^2)
    static constexpr int s = DEF ? 6 : 3;
    static constexpr uint32_t oinv = inv32(o);
};
static_assert(Den<false>::o << Den<false>::s == 360u && (uint64_t)Den<true>::o << Den<true>::s == 129600u, "D");
static_assert(Den<true>::oinv * 2025u == 1u, "2-adic inverse");
template <uint32_t O> struct Pw {
    uint32_t p[40];     // 2^(32 i) mod O, i = 0..39
    uint32_t ip[2];     // 2^(-32 L) mod O for L = 36, 37
    uint32_t ps[NSEG];  // 2^(32 p_s) mod O, p_s = seg0(s)
    uint32_t ips[NSEG]; // 2^(-32 p_s) mod O
};
template <uint32_t O> __host__ __device__ constexpr Pw<O> make_pw() {
    Pw<O> t{};
    for (int i = 0; i < 40; ++i) t.p[i] = modpow32(O, i);
    t.ip[0] = invmod(modpow32(O, 36), O);
    t.ip[1] = invmod(modpow32(O, 37), O);
    for (int i = 0; i < NSEG; ++i) {
        t.ps[i] = modpow32(O, seg0(i));
        t.ips[i] = invmod(modpow32(O, seg0(i)), O);
    }
    return t;
}
}  // namespace cls

__constant__ cls::Pw<45u> tg_cls_pw45 = cls::make_pw<45u>();
__constant__ cls::Pw<2025u> tg_cls_pw2025 = cls::make_pw<2025u>();
template <bool DEF> __device__ __forceinline__ const cls::Pw<cls::Den<DEF>::o>& cls_pw();
template <> __device__ __forceinline__ const cls::Pw<45u>& cls_pw<false>() { return tg_cls_pw45; }
template <> __device__ __forceinline__ const cls::Pw<2025u>& cls_pw<true>() { return tg_cls_pw2025; }

__host__ __device__ constexpr size_t cls_smem_bytes() {
    return (size_t)4 * ((size_t)cls::NP * cls::YW * cls::G + 4 * cls::NSEG * cls::G + cls::G);
}

// smem word offset (without the lane) of the lo word / packed high word of X[P]
__device__ __forceinline__ int cls_lo(int P) {
    const int m = P >> 6, r = P & 63;
    return (m <= 6 ? m * cls::YW + r : (m == 7 ? r + 64 : cls::YW + r + 64)) * cls::G;
}
__device__ __forceinline__ int cls_hi(int P) { return ((2 + (P >> 7)) * cls::YW + (P & 63) + 64) * cls::G; }

template <int J, int K>
__device__ __forceinline__ void cls_term(uint32_t y, uint64_t& p, uint64_t& n) {
    constexpr long long A = tg_combA_cx_T4(J, K);
    if constexpr (A > 0) p = tg_madw((uint32_t)A, y, p);
    else if constexpr (A < 0) n = tg_madw((uint32_t)(-A), y, n);
}
template <int J>
__device__ __forceinline__ void cls_row(const uint32_t (&y)[7], uint64_t& p, uint64_t& n) {
    cls_term<J, 0>(y[0], p, n);
    cls_term<J, 1>(y[1], p, n);
    cls_term<J, 2>(y[2], p, n);
    cls_term<J, 3>(y[3], p, n);
    cls_term<J, 4>(y[4], p, n);
    cls_term<J, 5>(y[5], p, n);
    cls_term<J, 6>(y[6], p, n);
}
// column t = r + 64 I of the products into X[r + 64 (I + j)]
template <int I>
__device__ __forceinline__ void cls_column(const uint32_t (&y)[7], uint64_t (&aP)[9], uint64_t (&aN)[9]) {
    cls_row<0>(y, aP[I], aN[I]);
    cls_row<1>(y, aP[I + 1], aN[I + 1]);
    cls_row<2>(y, aP[I + 2], aN[I + 2]);
    if constexpr (I + 3 <= 8) cls_row<3>(y, aP[I + 3], aN[I + 3]);
    if constexpr (I + 4 <= 8) cls_row<4>(y, aP[I + 4], aN[I + 4]);
    if constexpr (I + 5 <= 8) cls_row<5>(y, aP[I + 5], aN[I + 5]);
    if constexpr (I + 6 <= 8) cls_row<6>(y, aP[I + 6], aN[I + 6]);
}

// the class sums on the FP64 pipe (TG_CLS_FP64, default; as the bottom's,
// csrc/fused_dc.cuh): y < 2^32 and |A'_jk| <= 720 < 2^10 give terms below
// 2^42 and |X| < 2^45 (each accumulator sums at most 21 of them), so every
// DFMA result is an integer below 2^53, exact; the IMAD pipe is left to the
// division and carry phases of the other resident CTA
#ifndef TG_CLS_FP64
#define TG_CLS_FP64 1
#endif
template <int J>
__device__ __forceinline__ void cls_drow(const double (&y)[7], double& a) {
#pragma unroll
    for (int k = 0; k < 7; ++k) {
        const long long A = tg_combA_cx_T4(J, k);
        if (A != 0) a = fma((double)A, y[k], a);
    }
}
template <int I, int J = 0>
__device__ __forceinline__ void cls_dcolumn(const double (&y)[7], double (&a)[9]) {
    if constexpr (J < 7 && I + J <= 8) {
        cls_drow<J>(y, a[I + J]);
        cls_dcolumn<I, J + 1>(y, a);
    }
}
static_assert(21.0 * 720.0 * 4294967295.0 < 2251799813685248.0, "class sums below 2^51: exact in doubles and dc_d2ll");

__device__ __forceinline__ void cls_class_fp64(int r, uint32_t* Y, int lane) {
    using namespace cls;
    double a[9];
#pragma unroll
    for (int m = 0; m < 9; ++m) a[m] = 0.0;
    uint32_t* c0 = Y + r * G + lane;       // cells (k, r)
    uint32_t* c1 = c0 + 64 * G;            // cells (k, r + 64)
    {
        double y[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) y[k] = dc_u2d(c0[k * YW * G]);
        cls_dcolumn<0>(y, a);
    }
    {
        double y[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) y[k] = dc_u2d(c1[k * YW * G]);
        cls_dcolumn<1>(y, a);
    }
    if (r < 2) {            // t = r + 128 (columns 128, 129: never overwritten)
        double y[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) y[k] = dc_u2d(c1[(k * YW + 64) * G]);
        cls_dcolumn<2>(y, a);
    } else if (r == 2) {    // t = 130: y_k = -s_k, the sign of limb 129
        double y[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) y[k] = -(double)(Y[(k * YW + YW - 1) * G + lane] >> 31);
        cls_dcolumn<2>(y, a);
    }
    uint32_t hw[9];
#pragma unroll
    for (int m = 0; m < 9; ++m) {
        const uint64_t x = (uint64_t)dc_d2ll(a[m]);
        hw[m] = (uint32_t)(x >> 32) & 0xFFFFu;
        if (m <= 6) c0[m * YW * G] = (uint32_t)x;
        else if (m == 7) c1[0] = (uint32_t)x;
        else if (r == 0) c1[YW * G] = (uint32_t)x;   // P = 512
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) c1[(2 + h) * YW * G] = hw[2 * h] | (hw[2 * h + 1] << 16);
    if (r == 0) c1[6 * YW * G] = hw[8];
}

__device__ __forceinline__ void cls_class(int r, uint32_t* Y, int lane) {
    if constexpr (TG_CLS_FP64) {
        cls_class_fp64(r, Y, lane);
        return;
    }
    using namespace cls;
    uint64_t aP[9], aN[9];
#pragma unroll
    for (int m = 0; m < 9; ++m) aP[m] = aN[m] = 0ull;
    uint32_t* c0 = Y + r * G + lane;       // cells (k, r)
    uint32_t* c1 = c0 + 64 * G;            // cells (k, r + 64)
    {
        uint32_t y[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) y[k] = c0[k * YW * G];
        cls_column<0>(y, aP, aN);
    }
    {
        uint32_t y[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) y[k] = c1[k * YW * G];
        cls_column<1>(y, aP, aN);
    }
    if (r < 2) {            // t = r + 128 (columns 128, 129: never overwritten)
        uint32_t y[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) y[k] = c1[(k * YW + 64) * G];
        cls_column<2>(y, aP, aN);
    } else if (r == 2) {    // t = 130: y_k = -s_k, the sign of limb 129
        uint32_t sg[7];
#pragma unroll
        for (int k = 0; k < NP; ++k) sg[k] = Y[(k * YW + YW - 1) * G + lane] >> 31;
        cls_column<2>(sg, aN, aP);
    }
    // X[r + 64 m]: lo words in (m, r) (m = 7: (0, r + 64), m = 8: (1, r + 64)),
    // high words packed two per cell in (2 + m/2, r + 64)
    uint32_t hw[9];
#pragma unroll
    for (int m = 0; m < 9; ++m) {
        const uint64_t x = aP[m] - aN[m];
        hw[m] = (uint32_t)(x >> 32) & 0xFFFFu;
        if (m <= 6) c0[m * YW * G] = (uint32_t)x;
        else if (m == 7) c1[0] = (uint32_t)x;
        else if (r == 0) c1[YW * G] = (uint32_t)x;   // P = 512
    }
#pragma unroll
    for (int h = 0; h < 4; ++h) c1[(2 + h) * YW * G] = hw[2 * h] | (hw[2 * h + 1] << 16);
    if (r == 0) c1[6 * YW * G] = hw[8];
}

// runs of constant m = P / 64 inside a segment: lo words at stride G from
// cls_lo, packed highs (half m & 1) at stride G from cls_hi
template <bool HALF>
__device__ __forceinline__ void cls_carry_run(uint32_t* pl, const uint32_t* ph, const uint32_t* pw, int n,
                                              long long& carry, uint64_t& rho) {
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
        const uint32_t h = ph[i * cls::G];
        const int32_t hs = HALF ? ((int32_t)h >> 16) : ((int32_t)(h << 16) >> 16);
        const long long x = (long long)(((unsigned long long)(uint32_t)hs << 32) | pl[i * cls::G]) + carry;
        const uint32_t z = (uint32_t)x;
        carry = x >> 32;
        pl[i * cls::G] = z;
        rho += (uint64_t)z * pw[i];   // < 74 * 2^43
    }
}
template <uint32_t O, uint32_t OINV>
__device__ __forceinline__ void cls_div_run(uint32_t* pl, int n, uint32_t& bor) {
#pragma unroll 4
    for (int i = 0; i < n; ++i) {
        // one limb of the 2-adic exact division (ref [4]): q = (t - bor) o^-1,
        // bor' = hi(q o) + (t < bor)
        const uint32_t t = pl[i * cls::G];
        const uint32_t q = (t - bor) * OINV;
        bor = __umulhi(q, O) + (t < bor ? 1u : 0u);
        pl[i * cls::G] = q;
    }
}

template <bool DEF>
__global__ void __launch_bounds__(32 * cls::NW, 2) k_interp_top_cls(const uint32_t* __restrict__ P1, uint32_t* __restrict__ w,
                                                          size_t count) {
    using namespace cls;
    constexpr uint32_t o = Den<DEF>::o, oinv = Den<DEF>::oinv;
    constexpr int S = Den<DEF>::s;
    extern __shared__ uint32_t sm[];
    uint32_t* Y = sm;                          // [7][130][28] products, then X / z / q (class cells)
    uint32_t* ZL = Y + NP * YW * G;            // [7][28] segment limb 0 (carry-in 0)
    uint32_t* CO = ZL + NSEG * G;              //         segment carry-out (signed)
    uint32_t* RH = CO + NSEG * G;              //         segment residue of X mod o
    uint32_t* BI = RH + NSEG * G;              //         segment borrow-in
    uint32_t* FL = BI + NSEG * G;              // [28] a limb 0 wrapped (serial fix-up)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t c0 = (size_t)blockIdx.x * G;
    const int nin = (int)min((size_t)G, count - c0);
    const size_t SK = (size_t)NP * count;
    const bool act = lane < G;
    if (threadIdx.x < G) FL[threadIdx.x] = 0u;   // (read after phase 3's barriers)

    // ---- 0: rows (k, t) of G contiguous words; row R = t * 7 + k in source
    // order, 4 rows per warp instruction (7 lanes x 16 bytes each), a warp's
    // rows keep their point k and advance t by 8
    {
        const bool v16 = ((count & 3) == 0) && ((((uintptr_t)P1) & 15) == 0);
        const int sub = lane / 7, q = lane - 7 * sub;
        constexpr int TS = 4 * NW / NP;   // limb rows per step
        static_assert(4 * NW == TS * NP, "rows per step: whole limb rows of all points");
        if (sub < 4) {
            const int R0 = warp * 4 + sub;
            const int k = R0 % NP;
            int t = R0 / NP;
            const int g = q * 4;
            const uint32_t* sr = P1 + (size_t)t * SK + (size_t)k * count + c0 + g;
            uint32_t* dr = Y + (size_t)(k * YW + t) * G + g;
            const size_t sstep = (size_t)TS * SK;
            if (v16 && g + 3 < nin) {
                unsigned d = (unsigned)__cvta_generic_to_shared(dr);
                for (; t < YW; t += TS, sr += sstep, d += 4u * TS * G)
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(sr));
            } else {
                for (; t < YW; t += TS, sr += sstep, dr += TS * G) {
#pragma unroll
                    for (int x = 0; x < 4; ++x) dr[x] = (g + x < nin) ? __ldg(sr + x) : 0u;
                }
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();

    // ---- 1: the classes of this warp
    if (act)
        for (int r = warp; r < BB; r += NW) cls_class(r, Y, lane);
    __syncthreads();

    // ---- 2: carries over segment `warp` (carry-in 0) and its residue mod o
    const int p0 = seg0(warp), L = seg0(warp + 1) - p0;
    if (act) {
        const auto& pw = cls_pw<DEF>();
        long long carry = 0;
        uint64_t rho = 0;
        for (int P = p0; P < p0 + L;) {
            const int n = min(p0 + L, (P | 63) + 1) - P;   // to the end of the run of m = P / 64
            uint32_t* pl = Y + cls_lo(P) + lane;
            const uint32_t* ph = Y + cls_hi(P) + lane;
            if (P & 64) cls_carry_run<true>(pl, ph, pw.p + (P - p0), n, carry, rho);
            else cls_carry_run<false>(pl, ph, pw.p + (P - p0), n, carry, rho);
            P += n;
        }
        const long long cm = carry % (long long)o;
        const uint32_t r = (uint32_t)(rho % o) + (uint32_t)(cm < 0 ? cm + o : cm) * pw.p[L];
        ZL[warp * G + lane] = Y[cls_lo(p0) + lane];
        CO[warp * G + lane] = (uint32_t)(int32_t)carry;
        RH[warp * G + lane] = r % o;
    }
    __syncthreads();

    // ---- 3: carry-ins and borrow-ins.  Warp s forms its own: the carry into
    // p_s is the previous segment's carry-out (a carry-in is absorbed by the
    // limbs unless it wraps limb 0, probability ~2^-17 per segment: then the
    // product goes through warp 0's serial chain), the borrow-in follows from
    // 2^(-32 p_s) sum_{s' < s} rho_s' 2^(32 p_s') mod o
    if (act) {
        const auto& pw = cls_pw<DEF>();
        const long long c = warp ? (long long)(int32_t)CO[(warp - 1) * G + lane] : 0ll;
        uint32_t acc = 0;   // < 13 * o^2 < 2^26
        for (int s = 0; s < warp; ++s) acc += RH[s * G + lane] * pw.ps[s];
        const uint32_t T = (acc % o) * pw.ips[warp] % o;
        const long long cm = c % (long long)o;
        BI[warp * G + lane] = ((uint32_t)(cm < 0 ? cm + o : cm) + o - T) % o;
        const long long x = (long long)ZL[warp * G + lane] + c;
        Y[cls_lo(p0) + lane] = (uint32_t)x;
        if ((x >> 32) != 0 || tg_fault == 2) FL[lane] = 1u;   // (kind 2: tests take the serial chain)
    }
    __syncthreads();
    if (warp == 0 && act && FL[lane]) {
        const auto& pw = cls_pw<DEF>();
        long long c = 0;
        uint32_t T = 0;   // 2^(-32 p_s) sum_{i < p_s} X_i 2^(32 i) mod o
#pragma unroll 1
        for (int s = 0; s < NSEG; ++s) {
            const int ps = seg0(s), Ls = seg0(s + 1) - ps;
            const long long cm = c % (long long)o;
            BI[s * G + lane] = ((uint32_t)(cm < 0 ? cm + o : cm) + o - T) % o;
            const long long x = (long long)ZL[s * G + lane] + c;
            Y[cls_lo(ps) + lane] = (uint32_t)x;
            long long d = x >> 32;   // -1, 0, +1
            for (int i = 1; i < Ls && d != 0; ++i) {   // rare: limb 0 wrapped
                uint32_t* p = Y + cls_lo(ps + i) + lane;
                const uint32_t v = *p, nv = v + (uint32_t)d;
                *p = nv;
                d = (d > 0) ? (nv == 0u ? 1 : 0) : (v == 0u ? -1 : 0);
            }
            c = (long long)(int32_t)CO[s * G + lane] + d;
            T = (uint32_t)(((T + RH[s * G + lane]) % o) * (uint32_t)pw.ip[Ls == 36 ? 0 : 1] % o);
        }
    }
    __syncthreads();

    // ---- 4: the exact division of segment `warp` from its borrow-in
    if (act) {
        uint32_t bor = BI[warp * G + lane];
        for (int P = p0; P < p0 + L;) {
            const int n = min(p0 + L, (P | 63) + 1) - P;
            cls_div_run<o, oinv>(Y + cls_lo(P) + lane, n, bor);
            P += n;
        }
        if (tg_check_on) {
            if (warp == 0) tg_check_low(Y[lane], S);                 // exact 2^S: q_0's low bits
            if (warp == NSEG - 1 && bor != 0u) tg_flag_inexact();   // X >= 0: exact iff the last borrow is 0
        }
    }
    __syncthreads();

    // ---- 5: w = q >> S, row-major, 4 limbs per 16-byte store; group g
    // (limbs 4g..4g+3) reads q_{4g..4g+4}, consecutive cells inside a run of m
    if (act && lane < nin) {
        uint32_t* row = w + (c0 + lane) * (size_t)WOUT;
        const bool v4 = (((uintptr_t)w) & 15) == 0;
#pragma unroll 1
        for (int g = warp; g < WOUT / 4; g += NW) {
            const int P = 4 * g;
            const uint32_t* pq = Y + cls_lo(P) + lane;
            uint32_t q[5];
#pragma unroll
            for (int x = 0; x < 4; ++x) q[x] = pq[x * G];
            q[4] = ((P + 4) & 63) ? pq[4 * G] : Y[cls_lo(P + 4) + lane];
            uint32_t o4[4];
#pragma unroll
            for (int x = 0; x < 4; ++x) o4[x] = __funnelshift_r(q[x], q[x + 1], S);
            if (v4) *reinterpret_cast<uint4*>(row + P) = make_uint4(o4[0], o4[1], o4[2], o4[3]);
            else
#pragma unroll
                for (int x = 0; x < 4; ++x) row[P + x] = o4[x];
        }
    }
}

}  // namespace tg
