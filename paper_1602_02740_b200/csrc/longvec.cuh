// Long-vector (limb-parallel) executor for the upper recursion levels of a
// single large product (BASELINE configs C4, C5): few instances, long
// operands.  SURVEY.md §7 H1/H2, DESIGN.md §6.
//
// Every evaluation (step a2), interpolation (step a4) and recomposition
// (step a5) step of such a level is a sequence of OPS
//
//     dst = ((sum_i m_i * (S_i << s_i)) / o) >> shr        (o odd, all exact)
//
// over whole vectors, computed modulo 2^(32 W) (W = output limbs).  S_i is a
// slice of a source vector (limbs [start, start+len), zero- or sign-extended
// past len), which covers the block split of Eq. 1.1 (start = j b), the
// recomposition w = sum_j w_j 2^(32 b j) of Eq. 1.3 (s_i = 32 b j) and the
// generated evaluation / interpolation programs (gen/toomgen.py,
// emit_long_tables: the paper's even-odd + listing programs, PAPER.md:114-120,
// 154-158, 164-186, or their per-coefficient matrix form).
//
// One launch per op, one pass over the data: a tile of NT threads x CH limbs
// forms the linear combination limb by limb (64- or 128-bit accumulators),
// normalises it locally, and resolves the carries and the exact-division
// borrows across the whole vector with a single-pass decoupled look-back scan.
// The scan state between limb positions is (c, beta): c the signed carry of
// the linear combination, beta the 2-adic division borrow; a chunk maps it by
//     c'    = cout[p]                         p = piece(c) in {0,1,2}
//     beta' = beta*m - c*m + g[p]  (mod o)
// (p selects whether the chunk's low limbs absorb the incoming carry with a
// borrow/carry out of the chunk; the borrow follows from the closed form
// beta_t = -(x mod 2^(32t)) 2^(-32t) mod o).  These maps compose, so tiles
// publish their aggregate before their predecessors finish.
#pragma once

namespace tg {

#ifndef TG_LONGOP_MINB
#define TG_LONGOP_MINB 2   // two tiles per SM (<= 128 registers)
#endif
constexpr int LV_MAXT = 64;     // terms per op (the P32 recomposition has 63)
constexpr int LV_NT = 256;      // threads per tile
constexpr int LV_CH = 16;       // limbs per thread (long vectors; 4 for short ones)
constexpr int LV_TL = LV_NT * LV_CH;
constexpr int LV_MAXHALO = 10;  // look-ahead limbs of the final right shift (shr < 32*9: P32 shifts up to 271 bits)

struct LTermDev {
    const uint32_t* base;       // limb `start` of instance 0
    long long inst_stride;      // limbs between instances
    long long limb_stride;      // limbs between consecutive limbs of one value
    int len;                    // slice length; limbs >= len are the fill
    int sign;                   // 1: sign-extend past len, 0: zero-extend
    int a, r;                   // left shift by 32 a + r bits (0 <= r < 32)
    long long m;                // multiplier
};

struct __align__(16) LOpDev {
    uint32_t* dst;
    long long dst_inst_stride, dst_limb_stride;
    int W;                      // output limbs
    int nt;
    uint32_t o, oinv;           // exact division by odd o (o = 1: none)
    uint32_t p32, Mch, mi;      // 2^32 mod o, 2^(32 CH) mod o, (2^(32 CH))^-1 mod o
    unsigned long long orcp;    // floor(2^64 / o) (Barrett reduction)
    int sa, sr;                 // final right shift shr = 32 sa + sr
    int tiles_per_inst;
    int nthreads;               // threads per tile (multiple of 32, <= LV_NT)
    int ch;                     // limbs per thread (4 or 16)
    int count;
    int wide;                   // 128-bit accumulators
    LTermDev t[LV_MAXT];
};

struct LAgg {
    long long lo, hi;           // piece thresholds: p = 0 if c < lo, 2 if c >= hi, else 1
    long long cout[3];
    uint32_t m, g[3];
};

struct LStatus {
    unsigned flag;              // epoch*4 + {1 aggregate, 2 inclusive}
    unsigned beta;
    long long c;
    LAgg agg;
};

// modulus o (odd, < 2^32) with its Barrett reciprocal floor(2^64 / o)
struct LMod {
    uint32_t o;
    unsigned long long rcp;
};
__device__ __forceinline__ uint32_t lv_mod(unsigned long long x, const LMod& M) {
    if (M.o < 32768u && x < 0x100000000ull) {
        // 32-bit Barrett: rcp32 = floor((2^32 - 1) / o) derived from the 64-bit one
        const uint32_t x32 = (uint32_t)x, r32 = (uint32_t)(M.rcp >> 32);
        uint32_t r = x32 - __umulhi(x32, r32) * M.o;
        while (r >= M.o) r -= M.o;
        return r;
    }
    const unsigned long long q = __umul64hi(x, M.rcp);
    unsigned long long r = x - q * M.o;
    while (r >= M.o) r -= M.o;
    return (uint32_t)r;
}
__device__ __forceinline__ uint32_t lv_mulmod(uint32_t a, uint32_t b, const LMod& M) {
    return lv_mod((unsigned long long)a * b, M);
}
// (-c) mod o for a signed 64-bit c
__device__ __forceinline__ uint32_t lv_negmod(long long c, const LMod& M) {
    const uint32_t r = lv_mod((unsigned long long)(c < 0 ? -c : c), M);   // |c| mod o (|c| < 2^63)
    return c < 0 ? r : (r ? M.o - r : 0u);
}
__device__ __forceinline__ int lv_piece(const LAgg& A, long long c) { return c < A.lo ? 0 : (c >= A.hi ? 2 : 1); }
// element p of a 3-array without dynamic indexing (keeps it in registers)
template <typename T>
__device__ __forceinline__ T lv_sel(const T (&a)[3], int p) { return p == 0 ? a[0] : (p == 1 ? a[1] : a[2]); }

// A then B
__device__ __forceinline__ LAgg lv_compose(const LAgg& A, const LAgg& B, const LMod& M) {
    const uint32_t o = M.o;
    LAgg C;
    C.lo = A.lo;
    C.hi = A.hi;
    C.m = (o > 1) ? lv_mulmod(A.m, B.m, M) : 0u;
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        const long long c1 = A.cout[p];
        const int q = lv_piece(B, c1);
        C.cout[p] = lv_sel(B.cout, q);
        if (o > 1) {
            // (g + (-c) mod o) reduced before the multiply: (o-1) m + g < o^2 + o < 2^64
            uint32_t t = A.g[p] + lv_negmod(c1, M);
            if (t < A.g[p] || t >= o) t -= o;
            const unsigned long long x = (unsigned long long)t * B.m + lv_sel(B.g, q);
            C.g[p] = lv_mod(x, M);
        } else {
            C.g[p] = 0;
        }
    }
    return C;
}

__device__ __forceinline__ void lv_apply(const LAgg& A, long long& c, uint32_t& beta, const LMod& M) {
    const int p = lv_piece(A, c);
    if (M.o > 1) {
        uint32_t t = beta + lv_negmod(c, M);   // both < o < 2^32: reduce before the multiply
        if (t < beta || t >= M.o) t -= M.o;
        const unsigned long long x = (unsigned long long)t * A.m + lv_sel(A.g, p);
        beta = lv_mod(x, M);
    }
    c = lv_sel(A.cout, p);
}

__device__ __forceinline__ LAgg lv_shfl_up(const LAgg& a, int d) {
    LAgg r;
    r.lo = __shfl_up_sync(0xffffffffu, a.lo, d);
    r.hi = __shfl_up_sync(0xffffffffu, a.hi, d);
#pragma unroll
    for (int p = 0; p < 3; ++p) {
        r.cout[p] = __shfl_up_sync(0xffffffffu, a.cout[p], d);
        r.g[p] = __shfl_up_sync(0xffffffffu, a.g[p], d);
    }
    r.m = __shfl_up_sync(0xffffffffu, a.m, d);
    return r;
}

// limb i of slice S of term T for instance `inst` (i may be < 0 or >= len)
__device__ __forceinline__ uint32_t lv_slice(const LTermDev& T, const uint32_t* src, int i, uint32_t fill) {
    if (i < 0) return 0u;
    if (i >= T.len) return fill;
    return __ldg(src + (long long)i * T.limb_stride);
}

// accumulate sum_i m_i * limb_p(S_i << s_i) for positions p0 .. p0+N-1.
// A term whose slice starts above the chunk contributes nothing; one whose
// slice ended below it contributes the constant m * fill per limb.
template <typename Acc, int N>
__device__ __forceinline__ void lv_lincomb(const LOpDev& op, int nt, long long inst, int p0, Acc (&lin)[N]) {
    Acc cst = 0;
#pragma unroll
    for (int q = 0; q < N; ++q) lin[q] = 0;
    for (int k = 0; k < nt; ++k) {
        const LTermDev& T = op.t[k];
        const int i0 = p0 - T.a;
        if (i0 + N - 1 < 0) continue;
        const uint32_t* src = T.base + inst * T.inst_stride;
        uint32_t fill = 0;
        if (T.sign && T.len > 0) fill = (__ldg(src + (long long)(T.len - 1) * T.limb_stride) >> 31) ? 0xFFFFFFFFu : 0u;
        if (i0 - 1 >= T.len) {
            cst += (Acc)T.m * (Acc)fill;
            continue;
        }
        uint32_t v[N + 1];
#pragma unroll
        for (int q = 0; q <= N; ++q) v[q] = lv_slice(T, src, i0 - 1 + q, fill);
        const long long m = T.m;
#pragma unroll
        for (int q = 0; q < N; ++q) {
            const uint32_t x = T.r ? __funnelshift_l(v[q], v[q + 1], T.r) : v[q + 1];
            lin[q] += (Acc)m * (Acc)x;
        }
    }
#pragma unroll
    for (int q = 0; q < N; ++q) lin[q] += cst;
}

// Parameters of the carry/borrow scan and the final division + shift + store
// of one output of one tile (shared by k_long_op and k_long_eval).
struct LFinish {
    uint32_t oinv, p32, Mch, mi;
    int sa, sr, W;
    LStatus* st_base;          // status of tile j at st_base + j * st_stride
    int st_stride;
    uint32_t* dst;             // this instance's output
    long long dst_limb_stride;
};

struct LTileSmem {
    LAgg wagg[LV_NT / 32];
    long long c;
    unsigned beta;
};

// local normalisation of the tile's linear combination, carry / borrow scan
// (warp shuffles + decoupled look-back), exact limbs, exact division, right
// shift, coalesced store.  lin: this thread's CH positions p0 = tstart + tid*CH.
// phase: 0 = single pass with the decoupled look-back; two-pass scan for long
// vectors of many tiles: 1 = publish the tile aggregate and stop (k_long_scan
// then writes every tile's carry-in / borrow-in), 2 = read the tile's in-state
// and finish.
template <typename Acc, int CH, class HaloF>
__device__ __forceinline__ void lv_finish(const Acc (&lin)[CH], const LMod& M, const LFinish& P, unsigned epoch,
                                          unsigned tile, int k, int tstart, LTileSmem& sh, uint32_t* Q, HaloF halo_fn,
                                          int phase = 0) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5, TL = NT * CH;
    const uint32_t o = M.o;
    LAgg* s_wagg = sh.wagg;
    long long& s_c = sh.c;
    unsigned& s_beta = sh.beta;
    // local normalisation (carry-in 0) -> thread aggregate
    uint32_t x[CH];
    long long c = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const Acc v = lin[q] + (Acc)c;
        x[q] = (uint32_t)v;
        c = (long long)(v >> 32);
    }
    LAgg A;
    {
        const unsigned long long L64 = (unsigned long long)x[0] | ((unsigned long long)x[1] << 32);
        bool tz = true, to = true;
#pragma unroll
        for (int q = 2; q < CH; ++q) { tz &= (x[q] == 0u); to &= (x[q] == 0xFFFFFFFFu); }
        A.lo = (tz && L64 <= 0x8000000000000000ull) ? (long long)(0ull - L64) : LLONG_MIN;
        const unsigned long long comp = 0ull - L64;   // 2^64 - L64
        A.hi = (to && L64 != 0 && comp <= (unsigned long long)LLONG_MAX) ? (long long)comp : LLONG_MAX;
        A.cout[0] = c - 1;
        A.cout[1] = c;
        A.cout[2] = c + 1;
        if (o > 1) {
            uint32_t r = 0;
#pragma unroll
            for (int q = CH - 1; q >= 0; --q) r = lv_mod((unsigned long long)r * P.p32 + x[q], M);
            A.m = P.mi;
#pragma unroll
            for (int p = 0; p < 3; ++p) {
                // g[p] = (-Lmod + (p-1) M) * mi mod o
                unsigned long long t = (unsigned long long)(o - r) + (p == 2 ? P.Mch : 0u) + (p == 0 ? (o - P.Mch) : 0u);
                A.g[p] = lv_mulmod(lv_mod(t, M), P.mi, M);
            }
        } else {
            A.m = 0;
            A.g[0] = A.g[1] = A.g[2] = 0;
        }
    }
    // warp inclusive scan
    LAgg inc = A;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const LAgg prev = lv_shfl_up(inc, d);
        if (lane >= d) inc = lv_compose(prev, inc, M);
    }
    const LAgg excl = lv_shfl_up(inc, 1);   // valid for lane > 0
    if (lane == 31) s_wagg[warp] = inc;
    __syncthreads();
    // tile aggregate, published before the look-back
    const bool first = (k == 0);
    LStatus* st = P.st_base + (long long)tile * P.st_stride;
    if (phase == 1) {
        if (warp == 0 && lane == 0) {
            LAgg T = s_wagg[0];
            for (int w = 1; w < NW; ++w) T = lv_compose(T, s_wagg[w], M);
            st->agg = T;
        }
        return;
    }
    if (phase == 2) {
        if (tid == 0) {
            s_c = first ? 0 : st->c;
            s_beta = first ? 0u : st->beta;
        }
    } else if (warp == 0) {
        LAgg T = s_wagg[0];
        for (int w = 1; w < NW; ++w) T = lv_compose(T, s_wagg[w], M);
        long long cin = 0;
        uint32_t bin = 0;
        if (!first) {
            if (lane == 0) {
                st->agg = T;
                __threadfence();
                atomicExch(&st->flag, epoch * 4u + 1u);
            }
            // decoupled look-back over the tiles of this instance, a window
            // of 32 predecessors per step (lane L looks at tile jhi - L)
            const long long base = (long long)tile - k;   // first tile of the instance (always inclusive)
            bool have = false;
            LAgg acc;                                       // composition of the later windows
            long long jhi = (long long)tile - 1;
            for (;;) {
                const long long j = jhi - lane;
                unsigned f = 0;
                LAgg a;
                a.lo = LLONG_MIN; a.hi = LLONG_MAX;
                a.cout[0] = a.cout[1] = a.cout[2] = 0; a.m = 1; a.g[0] = a.g[1] = a.g[2] = 0;
                long long ic = 0;
                unsigned ib = 0;
                if (j >= base) {
                    LStatus* ps = P.st_base + j * P.st_stride;
                    do { f = *(volatile unsigned*)&ps->flag; } while (f != epoch * 4u + 1u && f != epoch * 4u + 2u);
                    __threadfence();
                    if (f == epoch * 4u + 2u) {
                        ic = *(volatile long long*)&ps->c;
                        ib = *(volatile unsigned*)&ps->beta;
                    } else {
                        volatile LAgg* va = (volatile LAgg*)&ps->agg;
                        a.lo = va->lo; a.hi = va->hi;
                        a.cout[0] = va->cout[0]; a.cout[1] = va->cout[1]; a.cout[2] = va->cout[2];
                        a.m = va->m; a.g[0] = va->g[0]; a.g[1] = va->g[1]; a.g[2] = va->g[2];
                    }
                }
                const unsigned incm = __ballot_sync(0xffffffffu, f == epoch * 4u + 2u);
                const int lim = incm ? (__ffs(incm) - 1) : 32;   // lanes [0, lim) carry aggregates
                // ordered reduction of the aggregates of lanes [0, lim) into lane 0
                // (a higher lane is an earlier tile: combined = compose(x[L+d], x[L]))
#pragma unroll
                for (int d = 1; d < 32; d <<= 1) {
                    LAgg other;
                    other.lo = __shfl_down_sync(0xffffffffu, a.lo, d);
                    other.hi = __shfl_down_sync(0xffffffffu, a.hi, d);
#pragma unroll
                    for (int p = 0; p < 3; ++p) {
                        other.cout[p] = __shfl_down_sync(0xffffffffu, a.cout[p], d);
                        other.g[p] = __shfl_down_sync(0xffffffffu, a.g[p], d);
                    }
                    other.m = __shfl_down_sync(0xffffffffu, a.m, d);
                    if ((lane & (2 * d - 1)) == 0 && lane + d < lim) a = lv_compose(other, a, M);
                }
                if (incm) {
                    ic = __shfl_sync(0xffffffffu, ic, lim);
                    ib = __shfl_sync(0xffffffffu, ib, lim);
                    if (lane == 0) {
                        cin = ic;
                        bin = ib;
                        if (lim > 0) lv_apply(a, cin, bin, M);
                        if (have) lv_apply(acc, cin, bin, M);
                    }
                    break;
                }
                if (lane == 0) {
                    acc = have ? lv_compose(a, acc, M) : a;
                    have = true;
                }
                have = __shfl_sync(0xffffffffu, have, 0);
                jhi -= 32;
            }
        }
        if (lane == 0) {
            // inclusive state of this tile
            long long cout = cin;
            uint32_t bout = bin;
            lv_apply(T, cout, bout, M);
            st->c = cout;
            st->beta = bout;
            __threadfence();
            atomicExch(&st->flag, epoch * 4u + 2u);
            s_c = cin;
            s_beta = bin;
        }
    }
    __syncthreads();
    // this thread's carry-in / borrow-in
    long long cin = s_c;
    uint32_t bin = s_beta;
    for (int w = 0; w < warp; ++w) lv_apply(s_wagg[w], cin, bin, M);
    if (lane > 0) lv_apply(excl, cin, bin, M);
    // exact limbs, exact division, quotients to smem
    c = cin;
    uint32_t beta = bin;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const Acc v = lin[q] + (Acc)c;
        uint32_t xq = (uint32_t)v;
        c = (long long)(v >> 32);
        if (o > 1) xq = tg_divexact_step(xq, beta, P.oinv, o);
        Q[tid * CH + q] = xq;
    }
    const int halo = P.sa + (P.sr ? 1 : 0);
    if (tid == NT - 1 && halo > 0) {
        // quotient limbs just past the tile (the next tile's first limbs),
        // continuing this tile's carry / borrow chain
        Acc hl[LV_MAXHALO];
        halo_fn(hl);
#pragma unroll
        for (int h = 0; h < LV_MAXHALO; ++h) {
            if (h >= halo) break;
            const Acc v = hl[h] + (Acc)c;
            uint32_t xq = (uint32_t)v;
            c = (long long)(v >> 32);
            if (o > 1) xq = tg_divexact_step(xq, beta, P.oinv, o);
            Q[TL + h] = xq;
        }
    }
    __syncthreads();
    // right shift, coalesced stores
    uint32_t* dst = P.dst;
    for (int i = tid; i < TL; i += NT) {
        const int t = tstart + i;
        if (t >= P.W) break;
        const uint32_t lo = Q[i + P.sa];
        const uint32_t y = P.sr ? __funnelshift_r(lo, Q[i + P.sa + 1], P.sr) : lo;
        dst[(long long)t * P.dst_limb_stride] = y;
    }
}

template <bool WIDE, int CH>
__global__ void __launch_bounds__(LV_NT, TG_LONGOP_MINB) k_long_op(const LOpDev* __restrict__ opp, LStatus* __restrict__ status,
                                                   unsigned epoch, unsigned* __restrict__ tile_ctr, int phase) {
    using Acc = typename std::conditional<WIDE, __int128, long long>::type;
    // the op descriptor (terms included) is cached in shared memory
    __shared__ __align__(16) LOpDev s_op;
    {
        const int4* srcd = reinterpret_cast<const int4*>(opp);
        int4* dstd = reinterpret_cast<int4*>(&s_op);
        constexpr int NQ = (int)(sizeof(LOpDev) / 16);
        for (int i = threadIdx.x; i < NQ; i += blockDim.x) dstd[i] = __ldg(srcd + i);
    }
    const LOpDev& op = s_op;
    __shared__ unsigned s_tile;
    __shared__ LTileSmem s_sh;
    extern __shared__ uint32_t Q[];               // [NT * CH + halo] quotient limbs
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5, TL = NT * CH;   // NT: a multiple of 32, <= LV_NT
    // single pass: dynamic tile ids (the look-back needs its predecessors
    // scheduled); two-pass phases: the block index
    if (tid == 0) s_tile = phase ? blockIdx.x : atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const unsigned tile = s_tile;
    const long long inst = tile / op.tiles_per_inst;
    const int k = (int)(tile - inst * op.tiles_per_inst);
    const int tstart = k * TL;
    const int p0 = tstart + tid * CH;
    const uint32_t o = op.o;
    const LMod M{op.o, op.orcp};
    const int nt = op.nt;

    Acc lin[CH];
    (void)p0;
    // the linear combination, one term at a time: the tile's slice of the term
    // is loaded coalesced into shared memory (position i of the tile at
    // Sx[(i % CH)][i / CH], row pitch NT + 1: conflict-free reads), then every
    // thread accumulates its CH positions.  Terms whose slice lies entirely
    // above the tile are skipped, terms entirely past their slice add m * fill.
    {
        uint32_t* Sx = Q + TL + LV_MAXHALO + 1;   // [CH][NT + 1] (+1 row for position -1)
        const int NP1 = NT + 1;
        Acc cst = 0;
#pragma unroll
        for (int q = 0; q < CH; ++q) lin[q] = 0;
        for (int kk = 0; kk < nt; ++kk) {
            const LTermDev& T = op.t[kk];
            const int ilo = tstart - T.a - 1, ihi = tstart + TL - 1 - T.a;   // slice indices the tile needs
            if (ihi < 0) continue;
            const uint32_t* src = T.base + inst * T.inst_stride;
            uint32_t fill = 0;
            if (T.sign && T.len > 0) fill = (__ldg(src + (long long)(T.len - 1) * T.limb_stride) >> 31) ? 0xFFFFFFFFu : 0u;
            if (ilo >= T.len) {
                cst += (Acc)T.m * (Acc)fill;
                continue;
            }
            __syncthreads();   // previous term's reads done
            // Sx row CH holds position -1 of each thread's chunk's predecessor:
            // store slice index ilo + 1 + i at (i % CH, i / CH); index ilo at the extra slot
            {
                // positions tid + q*NT (all loads issued before the stores)
                uint32_t xv[CH];
                if (ilo + 1 >= 0 && ihi < T.len) {   // interior tile: no bounds checks
                    const uint32_t* sp = src + (long long)(ilo + 1 + tid) * T.limb_stride;
                    const long long step = (long long)NT * T.limb_stride;
#pragma unroll
                    for (int q = 0; q < CH; ++q) xv[q] = __ldg(sp + q * step);
                } else {
#pragma unroll
                    for (int q = 0; q < CH; ++q) {
                        const int idx = ilo + 1 + tid + q * NT;
                        xv[q] = idx < 0 ? 0u : (idx >= T.len ? fill : __ldg(src + (long long)idx * T.limb_stride));
                    }
                }
                if (tid == 0) {
                    const int idx = ilo;      // position tstart - 1
                    Sx[CH * NP1] = idx < 0 ? 0u : (idx >= T.len ? fill : __ldg(src + (long long)idx * T.limb_stride));
                }
#pragma unroll
                for (int q = 0; q < CH; ++q) {
                    const int pos = tid + q * NT;
                    Sx[(pos % CH) * NP1 + pos / CH] = xv[q];
                }
            }
            __syncthreads();
            const long long m = T.m;
            const int r = T.r;
            // previous limb of my chunk's first position
            uint32_t prev = tid ? Sx[(CH - 1) * NP1 + tid - 1] : Sx[CH * NP1];
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const uint32_t cur = Sx[q * NP1 + tid];
                const uint32_t x = r ? __funnelshift_l(prev, cur, r) : cur;
                lin[q] += (Acc)m * (Acc)x;
                prev = cur;
            }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) lin[q] += cst;
        __syncthreads();   // Sx / Q reuse below
    }

    lv_finish<Acc, CH>(lin, M, LFinish{op.oinv, op.p32, op.Mch, op.mi, op.sa, op.sr, op.W, status, 1,
                                        op.dst + inst * op.dst_inst_stride, op.dst_limb_stride},
                       epoch, tile, k, tstart, s_sh, Q,
                       [&](Acc (&hl)[LV_MAXHALO]) { lv_lincomb<Acc, LV_MAXHALO>(op, nt, inst, tstart + TL, hl); },
                       phase);
}

// two-pass scan, pass 2: one CTA per instance turns the tile aggregates into
// every tile's carry-in / borrow-in (status[tile].c / .beta).  Thread t owns a
// contiguous run of tiles; runs are composed with a warp scan and the warps'
// totals are chained by warp 0.
__global__ void __launch_bounds__(1024) k_long_scan(LStatus* __restrict__ status, int tiles_per_inst, uint32_t o,
                                                    unsigned long long orcp) {
    const LMod M{o, orcp};
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
    const long long base = (long long)blockIdx.x * tiles_per_inst;
    const int per = (tiles_per_inst + blockDim.x - 1) / blockDim.x;
    const int t0 = min(tid * per, tiles_per_inst), t1 = min(t0 + per, tiles_per_inst);
    bool has = false;
    LAgg A;
    A.lo = LLONG_MIN; A.hi = LLONG_MAX;
    A.cout[0] = A.cout[1] = A.cout[2] = 0; A.m = 1; A.g[0] = A.g[1] = A.g[2] = 0;
    for (int t = t0; t < t1; ++t) {
        const LAgg x = status[base + t].agg;
        A = has ? lv_compose(A, x, M) : x;
        has = true;
    }
    // warp inclusive scan (with identity flags)
    LAgg inc = A;
    bool ihas = has;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const LAgg prev = lv_shfl_up(inc, d);
        const bool phas = __shfl_up_sync(0xffffffffu, ihas, d);
        if (lane >= d && phas) {
            inc = ihas ? lv_compose(prev, inc, M) : prev;
            ihas = true;
        }
    }
    const LAgg excl = lv_shfl_up(inc, 1);
    const bool ehas = __shfl_up_sync(0xffffffffu, ihas, 1) && lane > 0;
    __shared__ LAgg wtot[32];
    __shared__ bool whas[32];
    __shared__ long long wc[32];
    __shared__ unsigned wb[32];
    if (lane == 31) { wtot[warp] = inc; whas[warp] = ihas; }
    __syncthreads();
    if (tid == 0) {
        long long c = 0;
        uint32_t b = 0;
        for (int w = 0; w < NW; ++w) {
            wc[w] = c;
            wb[w] = b;
            if (whas[w]) lv_apply(wtot[w], c, b, M);
        }
    }
    __syncthreads();
    long long c = wc[warp];
    uint32_t b = wb[warp];
    if (ehas) lv_apply(excl, c, b, M);
    for (int t = t0; t < t1; ++t) {
        LStatus* st = status + base + t;
        const LAgg x = st->agg;
        st->c = c;
        st->beta = b;
        lv_apply(x, c, b, M);
    }
}

// ------------------------------------------------------------------------
// Multi-output op: NO outputs that are linear combinations of the SAME NS
// source slices, out_o = ((sum_s m[o][s] src_s) / o_o) >> shr_o.  A tile
// stages its limb range of every source in shared memory once, then runs the
// carry / borrow scan of every output in turn (status entries tile*NO + o).
// Serves the evaluation of a long level (sources = the B blocks, outputs =
// the 2B-1 points, Eq. 1.1-1.2) and its interpolation rows (sources = the
// 2B-1 products, outputs = the coefficient rows w_j = (sum_k A_jk y_k)/D_j of
// the even-odd + listing program).
// ------------------------------------------------------------------------
constexpr int LM_MAXS = 16, LM_MAXO = 31, LM_HALO = 8;

struct LMSrc {
    const uint32_t* base;       // slice start of instance 0 (row-major: limb stride 1)
    long long is;               // limbs between instances
    int len, sign;
};
struct LMOut {
    uint32_t* dst;              // instance 0
    unsigned long long orcp;
    uint32_t o, oinv, p32, Mch, mi;
    int sa, sr;
};
struct __align__(16) LMultiDev {
    int ns, no, W, tiles_per_inst, nthreads, ch, count, wide;
    long long dst_is, dst_ls;
    LMSrc src[LM_MAXS];
    LMOut out[LM_MAXO];
    long long m[LM_MAXO][LM_MAXS];
};

template <bool WIDE, int CH>
__global__ void __launch_bounds__(LV_NT, TG_LONGOP_MINB) k_long_multi(const LMultiDev* __restrict__ dp, LStatus* __restrict__ status,
                                                      unsigned epoch, unsigned* __restrict__ tile_ctr) {
    using Acc = typename std::conditional<WIDE, __int128, long long>::type;
    __shared__ __align__(16) LMultiDev s_d;
    {
        const int4* srcd = reinterpret_cast<const int4*>(dp);
        int4* dstd = reinterpret_cast<int4*>(&s_d);
        constexpr int NQ = (int)(sizeof(LMultiDev) / 16);
        for (int i = threadIdx.x; i < NQ; i += blockDim.x) dstd[i] = __ldg(srcd + i);
    }
    __shared__ unsigned s_tile;
    __shared__ LTileSmem s_sh;
    extern __shared__ uint32_t dsm[];
    const int tid = threadIdx.x, NT = blockDim.x, TL = NT * CH, NP1 = NT + 1 + (LM_HALO + CH - 1) / CH;
    uint32_t* Q = dsm;                                  // [TL + halo]
    uint32_t* Sb = dsm + TL + LV_MAXHALO + 1;           // [ns][CH][NP1]: position i at (i % CH, i / CH)
    if (tid == 0) s_tile = atomicAdd(tile_ctr, 1u);
    __syncthreads();
    const LMultiDev& d = s_d;
    const unsigned tile = s_tile;
    const long long inst = tile / d.tiles_per_inst;
    const int kt = (int)(tile - inst * d.tiles_per_inst);
    const int tstart = kt * TL;
    // stage positions [tstart, tstart + TL + LM_HALO) of every source
    for (int sI = 0; sI < d.ns; ++sI) {
        const LMSrc& S = d.src[sI];
        const uint32_t* sp = S.base + inst * S.is;
        uint32_t fill = 0;
        if (S.sign && S.len > 0) fill = (__ldg(sp + (S.len - 1)) >> 31) ? 0xFFFFFFFFu : 0u;
        uint32_t* sj = Sb + (size_t)sI * CH * NP1;
        for (int i = tid; i < TL + LM_HALO; i += NT) {
            const int t = tstart + i;
            sj[(i % CH) * NP1 + i / CH] = (t < S.len) ? __ldg(sp + t) : fill;
        }
    }
    __syncthreads();
    for (int o = 0; o < d.no; ++o) {
        const LMOut& O = d.out[o];
        Acc lin[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) lin[q] = 0;
        for (int sI = 0; sI < d.ns; ++sI) {
            const long long m = d.m[o][sI];
            if (m == 0) continue;
            const uint32_t* sj = Sb + (size_t)sI * CH * NP1 + tid;
#pragma unroll
            for (int q = 0; q < CH; ++q) lin[q] += (Acc)m * (Acc)sj[q * NP1];
        }
        const LMod M{O.o, O.orcp};
        lv_finish<Acc, CH>(lin, M, LFinish{O.oinv, O.p32, O.Mch, O.mi, O.sa, O.sr, d.W, status + o, d.no,
                                           O.dst + inst * d.dst_is, d.dst_ls},
                           epoch, tile, kt, tstart, s_sh, Q, [&](Acc (&hl)[LV_MAXHALO]) {
                               // positions TL .. TL + LV_MAXHALO - 1 from the staged halo
#pragma unroll
                               for (int h = 0; h < LV_MAXHALO; ++h) {
                                   Acc v = 0;
                                   const int i = TL + h;
                                   for (int s2 = 0; s2 < d.ns; ++s2)
                                       v += (Acc)d.m[o][s2] * (Acc)Sb[(size_t)s2 * CH * NP1 + (i % CH) * NP1 + i / CH];
                                   hl[h] = v;
                               }
                           });
    }
}

inline size_t long_multi_smem(int nthreads, int ch, int ns) {
    const int np1 = nthreads + 1 + (LM_HALO + ch - 1) / ch;
    return 4 * ((size_t)nthreads * ch + LV_MAXHALO + 1 + (size_t)ns * ch * np1);
}

// ------------------------------------------------------------------------
// host side: op builder
// ------------------------------------------------------------------------
struct LVec {                  // a vector family: value of instance c, limb i at base[c*is + i*ls]
    const uint32_t* base;
    long long is, ls;
    int len;                   // exact length (limbs beyond: fill)
    int sign;
};

static uint32_t host_inv32(uint32_t o) {
    uint32_t x = o;            // Newton: x = x (2 - o x), 5 steps from 3 bits
    for (int i = 0; i < 5; ++i) x *= 2u - o * x;
    return x;
}
static uint32_t host_powmod(unsigned long long b, unsigned long long e, uint32_t o) {
    unsigned long long r = 1 % o;
    b %= o;
    while (e) {
        if (e & 1) r = r * b % o;
        b = b * b % o;
        e >>= 1;
    }
    return (uint32_t)r;
}
static uint32_t host_invmod(uint32_t a, uint32_t o) {   // o odd, gcd(a, o) = 1
    long long t = 0, nt = 1, r = o, nr = a % o;
    while (nr) {
        long long q = r / nr;
        long long x = t - q * nt; t = nt; nt = x;
        x = r - q * nr; r = nr; nr = x;
    }
    if (t < 0) t += o;
    return (uint32_t)t;
}

// set when an op needed more than LV_MAXT terms; the call that built it fails
inline bool& lv_build_overflow() {
    static thread_local bool f = false;
    return f;
}

struct LOpBuilder {
    LOpDev op;
    LOpBuilder(uint32_t* dst, long long is, long long ls, int W, int count, uint32_t o = 1, int shr = 0) {
        memset(&op, 0, sizeof op);
        op.dst = dst;
        op.dst_inst_stride = is;
        op.dst_limb_stride = ls;
        op.W = W;
        op.count = count;
        op.o = o;
        op.oinv = host_inv32(o);
        // limbs per thread: 16 for long vectors, 4 for short ones; tile size:
        // the fewest padded limbs, then the largest tile
        op.ch = 16;   // the scan costs ~1k instructions per thread: amortise over 16 limbs
        // the largest tile that pads the vector by at most 1/8 (else the least padding)
        int best = LV_NT;
        long long bestw = -1;
        for (int nt = LV_NT; nt >= 32; nt -= 32) {
            const long long tl = (long long)nt * op.ch, tiles = (W + tl - 1) / tl;
            const long long pad = tiles * tl;
            if (pad * 8 <= (long long)W * 9) { best = nt; bestw = pad; break; }
            if (bestw < 0 || pad < bestw) { bestw = pad; best = nt; }
        }
        op.nthreads = best;
        op.tiles_per_inst = (W + best * op.ch - 1) / (best * op.ch);
        if (o > 1) {
            op.orcp = ~0ull / o;   // floor((2^64 - 1) / o) == floor(2^64 / o) for odd o > 1
            op.p32 = host_powmod(2, 32, o);
            op.Mch = host_powmod(2, 32ull * op.ch, o);
            op.mi = host_invmod(op.Mch, o);
        }
        op.sa = shr / 32;
        op.sr = shr % 32;
    }
    // term m * (slice << s), slice = limbs [start, start+len) of v (len clipped to v.len)
    bool add(const LVec& v, long long m, long long s, int start = 0, int len = -1, int sign = -1) {
        if (m == 0) return true;
        if (op.nt >= LV_MAXT) { lv_build_overflow() = true; return false; }   // the call fails (EUNSUPPORTED)
        LTermDev& T = op.t[op.nt++];
        T.base = v.base + (long long)start * v.ls;
        T.inst_stride = v.is;
        T.limb_stride = v.ls;
        const int avail = v.len - start;
        T.len = len < 0 ? avail : (len < avail ? len : avail);
        if (T.len < 0) T.len = 0;
        // a slice that stops inside the exact value is zero-extended unless asked
        T.sign = sign < 0 ? ((T.len == avail) ? v.sign : 0) : sign;
        T.a = (int)(s / 32);
        T.r = (int)(s % 32);
        T.m = m;
        return true;
    }
};

}  // namespace tg
