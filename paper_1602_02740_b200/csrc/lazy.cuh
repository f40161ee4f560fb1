// Lazy Toom-3/4 levels: the levels of a single large product (C4, and the
// Toom-4 levels under C5's Toom-16 top) from the top down to the fused bottom
// level, run without any carry propagation or division on the way.
//
// A lazy vector of W positions is two uint32 arrays LO, HI with
//     value = sum_p (LO[p] + HI[p]) 2^(32 p),   LO unsigned, HI signed (small),
// i.e. position p holds v_p = LO[p] + HI[p] with |v_p| < 2^33.  Every step of
// the method on these levels is linear in its inputs:
//   a2 evaluation   U(x_k)[t] = sum_j c_kj u_j[t]          (Eq. 1.1, 4.1)
//   a4+a5           Dc w = sum_j 2^(32 b j) N_j,  N_j = sum_k c'_jk y_k
//                   (the even-odd + listing program composed over the common
//                   denominator Dc = lcm D_j; DESIGN reading 12)
// so each is one elementwise pass: position p of the output is a linear form
// lin_p of input positions, stored as LO = lin_p mod 2^32 at p and
// HI = floor(lin_p / 2^32) at p + 1 (the carry is kept, not propagated).  The
// exact divisions are deferred: the products coming up from a lazy level carry
// the factor Dc of every lazy level below, and the division by
// prod Dc = 2^s o1 o2 .. (word factors) plus the carry propagation runs once at
// the top of the lazy block (k_lz_fin, the two-pass scan of longvec2.cuh).
// The deepest lazy level writes carry-normalised children (k_lz_eval_last),
// the input of the fused bottom level.
//
// Layout: every lazy family is INTERLEAVED, position p of row R at p*rows + R
// (row R = k*count + c for child k of parent c), and every kernel maps its
// linear thread index to (position, row) with the row fastest, so that all
// reads and writes of a warp are contiguous for any count (count = 1 is the
// row-major single product).
//
// Bounds: |v_p| < 2^32 + 2^31 on every lazy vector (|HI| < 2^17 below), the
// evaluation forms are < 15 * 2^33 < 2^37, the interpolation forms
// < 3 * 2520 * 2^33 < 2^47 (T4: row sums of |c'_jk| <= 2520): int64 throughout.
#pragma once

namespace tg {

// a family of vectors of n positions: position p of row r at r*is + p*ps
struct LzSrc {
    const uint32_t* lo;   // normalised limbs, or the LO array of a lazy family
    const uint32_t* hi;   // nullptr: normalised (two's complement if sgn)
    long long is, ps;     // row and position strides
    int n;                // positions per row
    int sgn;              // normalised rows: top limb signed
};

__device__ __forceinline__ long long lz_get(const LzSrc& S, long long row, int p) {
    if (p >= S.n) return 0;
    const long long o = row * S.is + (long long)p * S.ps;
    const uint32_t x = __ldg(S.lo + o);
    if (S.hi) return (long long)x + (long long)(int)__ldg(S.hi + o);
    return (S.sgn && p == S.n - 1) ? (long long)(int)x : (long long)x;
}

// g = q d + r for a linear thread index g (< 2^63) and the row count d, with
// dinv = floor((2^64 - 1) / d): one high multiply and one correction
__device__ __forceinline__ long long lz_div(long long g, long long d, unsigned long long dinv, long long& r) {
    unsigned long long q = __umul64hi((unsigned long long)g, dinv);
    long long rem = g - (long long)q * d;
    if (rem >= d) { ++q; rem -= d; }
    r = rem;
    return (long long)q;
}

// position p of row `row` in split form v = lo + hi + hs 2^32: hi the lazy
// carry of the position (same weight), hs the sign of a normalised top limb
__device__ __forceinline__ void lz_get2(const LzSrc& S, long long row, int p, uint32_t& lo, int& hi, int& hs) {
    lo = 0;
    hi = 0;
    hs = 0;
    if (p >= S.n) return;
    const long long o = row * S.is + (long long)p * S.ps;
    lo = __ldg(S.lo + o);
    if (S.hi) hi = (int)__ldg(S.hi + o);
    else if (S.sgn && p == S.n - 1) hs = -(int)(lo >> 31);
}

template <int B>
__device__ __forceinline__ constexpr long long lz_evalc(int k, int j) {
    if constexpr (B == 3) return tg_evalc_cx_T3(k, j);
    else return tg_evalc_cx_T4(k, j);
}
template <int B>
__device__ __forceinline__ constexpr long long lz_comb(int j, int k) {
    if constexpr (B == 3) return tg_combA_cx_T3(j, k);
    else return tg_combA_cx_T4(j, k);
}

// the 2B - 1 point values of one position from the blocks' values v_j
// (|v_j| < 2^34): Toom-4 with the +-x pairs sharing E = v0 + x^2 v2 and
// O = x v1 + x^3 v3 (Eqs. 4.3-4.4; the coefficients are powers of two, so
// shifts and adds); the generic form otherwise
template <int B>
__device__ __forceinline__ void lz_points(const long long (&v)[B], long long (&lin)[2 * B - 1]) {
    if constexpr (B == 4) {
        static_assert(tg_evalc_cx_T4(1, 1) == 1 && tg_evalc_cx_T4(2, 1) == -1 && tg_evalc_cx_T4(3, 3) == 8 &&
                          tg_evalc_cx_T4(4, 3) == -8 && tg_evalc_cx_T4(5, 0) == 8 && tg_evalc_cx_T4(6, 3) == 1,
                      "point order 0, 1, -1, 2, -2, 1/2 (homogeneous), inf");
        const long long E1 = v[0] + v[2], O1 = v[1] + v[3];
        const long long E2 = v[0] + v[2] * 4, O2 = v[1] * 2 + v[3] * 8;
        lin[0] = v[0];
        lin[1] = E1 + O1;
        lin[2] = E1 - O1;
        lin[3] = E2 + O2;
        lin[4] = E2 - O2;
        lin[5] = v[0] * 8 + v[1] * 4 + v[2] * 2 + v[3];
        lin[6] = v[3];
    } else {
#pragma unroll
        for (int k = 0; k < 2 * B - 1; ++k) {
            long long x = 0;
#pragma unroll
            for (int j = 0; j < B; ++j) x += lz_evalc<B>(k, j) * v[j];
            lin[k] = x;
        }
    }
}

// ---- a2: evaluation of one lazy level -------------------------------------
// child k of parent c at position t: lin = sum_j c_kj par_j[t], block j =
// parent positions [j b, j b + len_j); written to the interleaved lazy family
// (rows NP*count, e positions).  Thread g = t*count + c (blockIdx.y: operand).
template <int B>
__global__ void __launch_bounds__(256) k_lz_eval(LzSrc pu, LzSrc pv, uint32_t* __restrict__ ulo, uint32_t* __restrict__ uhi,
                                                 uint32_t* __restrict__ vlo, uint32_t* __restrict__ vhi, long long count,
                                                 unsigned long long cinv, int b, int lentop, int e) {
    constexpr int NP = 2 * B - 1;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long c;
    const long long t = lz_div(g, count, cinv, c);
    if (t >= e) return;
    const LzSrc& S = blockIdx.y ? pv : pu;
    uint32_t* lo = blockIdx.y ? vlo : ulo;
    uint32_t* hi = blockIdx.y ? vhi : uhi;
    long long v[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
        const int len = (j == B - 1) ? lentop : b;
        uint32_t xl = 0;
        int xh = 0, xs = 0;
        if (t < len) lz_get2(S, c, j * b + (int)t, xl, xh, xs);
        v[j] = (long long)xl + xh + ((long long)xs << 32);
    }
    long long lin[NP];
    lz_points<B>(v, lin);
    const long long rows = NP * count;
    uint32_t* pl = lo + t * rows + c;
    uint32_t* ph = hi + (t + 1) * rows + c;
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        pl[k * count] = (uint32_t)lin[k];
        if (t + 1 < e) ph[k * count] = (uint32_t)(int)(lin[k] >> 32);
        if (t == 0) hi[k * count + c] = 0u;
    }
}

// The same for the first level of a single product (COUNT parents): a warp's
// stores of one child are runs of `count` words 7 count apart (28 sectors
// per store at count = 1: the level was bound by the store path, 34 us for
// 38 MB, profiles/r02_c4_ncu_raw_summary.csv), so the CTA's outputs, one
// contiguous range of the family, are staged in shared memory and copied
// out in address order.
// (COUNT at compile time, 32-bit indices: the divisions of the copy-out by
// runtime values cost more than the stores saved, 24 -> 39 us at count = 7)
template <int B, int COUNT>
__global__ void __launch_bounds__(256) k_lz_eval_small(LzSrc pu, LzSrc pv, uint32_t* __restrict__ ulo, uint32_t* __restrict__ uhi,
                                                       uint32_t* __restrict__ vlo, uint32_t* __restrict__ vhi, int b,
                                                       int lentop, int e) {
    constexpr int NP = 2 * B - 1, NT = 256;
    constexpr unsigned count = COUNT, rows = NP * COUNT;
    constexpr int CAP = NP * (NT + 2 * COUNT);
    __shared__ uint32_t slo[CAP], shi[CAP];
    const unsigned g0 = blockIdx.x * NT;          // (e * count < 2^31: the host's launch condition)
    const unsigned g = g0 + threadIdx.x;
    const unsigned t = g / count, c = g - t * count;
    const unsigned t_first = g0 / count;
    const LzSrc& S = blockIdx.y ? pv : pu;
    uint32_t* lo = blockIdx.y ? vlo : ulo;
    uint32_t* hi = blockIdx.y ? vhi : uhi;
    if (t < (unsigned)e) {
        long long v[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const int len = (j == B - 1) ? lentop : b;
            uint32_t xl = 0;
            int xh = 0, xs = 0;
            if ((int)t < len) lz_get2(S, c, j * b + (int)t, xl, xh, xs);
            v[j] = (long long)xl + xh + ((long long)xs << 32);
        }
        long long lin[NP];
        lz_points<B>(v, lin);
        const unsigned r0 = (t - t_first) * rows + c;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            slo[r0 + k * count] = (uint32_t)lin[k];
            shi[r0 + k * count] = (uint32_t)(int)(lin[k] >> 32);
        }
    }
    __syncthreads();
    const unsigned t_last = (g0 + NT - 1) / count;
    const unsigned region = (t_last - t_first + 1) * rows;
    for (unsigned r = threadIdx.x; r < region; r += NT) {
        const unsigned tt = r / rows, rem = r - tt * rows;
        const unsigned cc = rem % count;
        const unsigned t2 = t_first + tt;
        const unsigned g2 = t2 * count + cc;
        if (g2 < g0 || g2 >= g0 + NT || t2 >= (unsigned)e) continue;
        lo[(size_t)t2 * rows + rem] = slo[r];
        if (t2 + 1 < (unsigned)e) hi[(size_t)(t2 + 1) * rows + rem] = shi[r];
        if (t2 == 0) hi[rem] = 0u;
    }
}

// ---- a2 of the deepest lazy level: evaluation + carry normalisation --------
// One thread per (parent, operand): the 2B-1 children position by position,
// each with its own carry chain, written as e two's-complement limbs to the
// interleaved family [e][NP*count] (the fused bottom level's MODE 0 input).
template <int B>
__global__ void __launch_bounds__(64, 25) k_lz_eval_last(LzSrc pu, LzSrc pv, uint32_t* __restrict__ du,
                                                      uint32_t* __restrict__ dv, long long count, int b, int lentop,
                                                      int e) {
    constexpr int NP = 2 * B - 1;
    const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    const LzSrc& S = blockIdx.y ? pv : pu;
    uint32_t* dst = (blockIdx.y ? dv : du) + c;
    const long long rows = NP * count;
    int cy[NP];   // |lin| < 2^37 (|c_kj| sums to <= 15, lazy carries small): carries fit 32 bits
#pragma unroll
    for (int k = 0; k < NP; ++k) cy[k] = 0;
    // (the even-odd sharing of lz_points measured slower here: 318 -> 341 us
    // on C4's deepest level, whose per-thread carry chains favour these
    // independent sums)
#pragma unroll 2
    for (int t = 0; t < e; ++t) {
        uint32_t xl[B];
        int xh[B], xs[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const int len = (j == B - 1) ? lentop : b;
            xl[j] = 0;
            xh[j] = 0;
            xs[j] = 0;
            if (t < len) lz_get2(S, c, j * b + t, xl[j], xh[j], xs[j]);
        }
        uint32_t* d = dst + (long long)t * rows;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            uint64_t P = 0, N = 0;
            int H = 0, Hs = 0;
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const long long m = lz_evalc<B>(k, j);
                if (m > 0) P += (uint64_t)m * xl[j];
                else if (m < 0) N += (uint64_t)(-m) * xl[j];
                if (m != 0) { H += (int)m * xh[j]; Hs += (int)m * xs[j]; }
            }
            const long long lin = (long long)cy[k] + (long long)(P - N) + (long long)H + ((long long)Hs << 32);
            d[k * count] = (uint32_t)lin;
            cy[k] = (int)(lin >> 32);
        }
    }
}

// ---- a4 + a5: interpolation and recomposition of one lazy level ------------
// X = Dc w = sum_j 2^(32 b j) N_j, N_j = sum_k c'_jk y_k; position P = s b + r
// receives N_{s-m}[m b + r] for every segment m of the products.  Thread
// g = r*count + c, r in [0, b): it reads y_k[m b + r] once for all m, k and
// writes the positions s b + r of the interleaved lazy output [Wx][count].
// Products of point k of parent c: row k*count + c of `y` (interleaved).
// Each term c'_jk (LO + HI) is one IMAD.WIDE.U32 into a positive or negative
// 64-bit accumulator (by the sign of the constant) plus a 32-bit MAD of HI.
template <int B, int MM, bool LZ>
__global__ void __launch_bounds__(256) k_lz_interp(LzSrc y, uint32_t* __restrict__ xlo, uint32_t* __restrict__ xhi,
                                                   long long count, unsigned long long cinv, int b, int Wx) {
    constexpr int NP = 2 * B - 1, NS = NP + MM - 1;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    long long c;
    const long long rr = lz_div(g, count, cinv, c);
    if (rr >= b) return;
    const int r = (int)rr;
    uint64_t Xp[NS], Xn[NS];
    int Xh[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) { Xp[s] = 0; Xn[s] = 0; Xh[s] = 0; }
    const long long ks = count * y.is, ms = (long long)b * y.ps;
    const uint32_t* ylo = y.lo + c * y.is + (long long)r * y.ps;
    const uint32_t* yhi = LZ ? y.hi + c * y.is + (long long)r * y.ps : nullptr;
#pragma unroll
    for (int m = 0; m < MM; ++m) {
        const int p = m * b + r;
        const bool in = m < MM - 1 || p < y.n;
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            const long long o = k * ks + m * ms;
            uint32_t lo = 0;
            int hi = 0;
            if (in) {
                lo = __ldg(ylo + o);
                if constexpr (LZ) hi = (int)__ldg(yhi + o);
            }
#pragma unroll
            for (int j = 0; j < NP; ++j) {
                const long long a = lz_comb<B>(j, k);
                if (a > 0) Xp[j + m] += (uint64_t)a * lo;
                else if (a < 0) Xn[j + m] += (uint64_t)(-a) * lo;
                if constexpr (LZ) { if (a != 0) Xh[j + m] += (int)a * hi; }
            }
        }
    }
    if constexpr (!LZ) {
        // normalised two's-complement products: the top limb (position n-1,
        // segment m = (n-1) / b) of a negative y_k weighs -2^32 more
        const int p = y.n - 1, m = p / b;
        if (y.sgn && p - m * b == r) {
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                const int neg = (int)(__ldg(ylo + k * ks + m * ms) >> 31);
#pragma unroll
                for (int mm = 0; mm < MM; ++mm)
                    if (mm == m) {
#pragma unroll
                        for (int j = 0; j < NP; ++j) Xh[j + mm] -= (int)lz_comb<B>(j, k) * neg;
                    }
            }
        }
    }
    uint32_t* ol = xlo + c + (long long)r * count;
    uint32_t* oh = xhi + c + (long long)(r + 1) * count;
    const long long sb = (long long)b * count;
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        const int P = s * b + r;
        if (P >= Wx) break;
        const long long X = (long long)(Xp[s] - Xn[s]) + (LZ ? (long long)Xh[s] : ((long long)Xh[s] << 32));
        ol[s * sb] = (uint32_t)X;
        if (P + 1 < Wx) oh[s * sb] = (uint32_t)(int)(X >> 32);
    }
    if (r == 0) xhi[c] = 0u;
}

// ---- normalisation + the deferred exact division (two-pass scan) ----------
// dst row c (Wout limbs, two's complement) = ((sum_p v_p 2^(32p)) / o) >> (32 sa + sr)
struct LzFin {
    LzSrc x;                   // lazy rows (or normalised)
    uint32_t* dst;
    long long dst_is;
    int Wout, tpi;
    long long rows;
    uint32_t o, oinv, p32, Mch, mi;
    int sa, sr;
};

template <int CH>
__global__ void __launch_bounds__(LV_NT, 4) k_lz_fin(LzFin F, LTile* __restrict__ tiles, int phase) {
    __shared__ L2Smem s_sh;
    extern __shared__ uint32_t Q[];
    const int tid = threadIdx.x, NT = blockDim.x, TL = NT * CH;
    // blocks position-major (the rows of one position range run together:
    // interleaved inputs share their sectors); tile records row-major
    const long long kt = blockIdx.x / F.rows;
    const long long inst = blockIdx.x - kt * F.rows;
    const unsigned tile = (unsigned)(inst * F.tpi + kt);
    const int tstart = (int)kt * TL;
    long long lin[CH];
    // reads at positions tstart + tid + q NT, transposed through smem to CH
    // consecutive positions per thread (two 32-bit halves)
    {
        const int NP1 = NT + 1;
        uint32_t* Sx = Q + lv2_qwords(TL, CH);
        long long xv[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) xv[q] = lz_get(F.x, inst, tstart + tid + q * NT);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            __syncthreads();
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int pos = tid + q * NT;
                Sx[(pos % CH) * NP1 + pos / CH] = h ? (uint32_t)(xv[q] >> 32) : (uint32_t)xv[q];
            }
            __syncthreads();
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const uint32_t w = Sx[q * NP1 + tid];
                if (h) lin[q] += (long long)(int)w << 32;
                else lin[q] = (long long)w;
            }
        }
        __syncthreads();
    }
    const LMod M{F.o, F.o > 1 ? ~0ull / F.o : 0ull};
    lv2_tile<long long, CH>(lin, M,
                            LFinish{F.oinv, F.p32, F.Mch, F.mi, F.sa, F.sr, F.Wout, reinterpret_cast<LStatus*>(tiles), 1,
                                    F.dst + inst * F.dst_is, 1},
                            tile, tstart, s_sh, Q,
                            [&](long long (&hl)[LV_MAXHALO]) {
#pragma unroll
                                for (int h = 0; h < LV_MAXHALO; ++h) hl[h] = lz_get(F.x, inst, tstart + TL + h);
                            },
                            phase);
}
inline size_t lz_fin_smem(int nthreads, int ch) {
    return 4 * ((size_t)lv2_qwords(nthreads * ch, ch) + (size_t)ch * (nthreads + 1));
}

}  // namespace tg
