// libtoomgpu: batched B-way Toom-Cook multiplication on B200 (sm_100a).
//
// Data path (DESIGN.md §"Kernels"):
//   level 0 eval   k_eval<PS, TOP=true>   row-major u, v -> child operands   (step a1+a2)
//   level l eval   k_eval<PS, TOP=false>  interleaved signed parents -> children
//   base case      k_base<E>              register-resident schoolbook         (step a3)
//   level l interp k_interp<PS, TOP>      2B-1 child products -> w_k -> parent (steps a4+a5)
// All intermediate values live in device memory in an INTERLEAVED layout:
// limb i of instance c of a level at [i * count + c], so that one thread per
// instance reads and writes fully coalesced across a warp.  Values below the
// top level are two's-complement integers (the evaluated values U(x_k) can
// be negative, Eq. 4.4).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <vector>
#include <mutex>
#include <string>
#include <climits>
#include <algorithm>
#include <type_traits>

#include "../../include/toomgpu.h"
#include "check.cuh"
#include "generated/toom_programs.cuh"

namespace tg {

// ------------------------------------------------------------------------
// point-set descriptors (the programs themselves are generated, see
// gen/toomgen.py).  ids: 0 = T3, 1 = T4, 2 = P8
// ------------------------------------------------------------------------
struct PSDesc {
    int B;
    int npts;
    uint64_t S;   // max over points of sum_k |p^k q^(n-k)| (value growth factor)
    int grow;     // limbs an evaluated operand grows by: e = b + grow
};

static int bitlen(uint64_t x) { int b = 0; while (x) { ++b; x >>= 1; } return b; }

static PSDesc ps_desc(int B) {
    auto g = [](uint64_t S) { return (bitlen(S) + 1 + 31) / 32; };
    switch (B) {
        case 3: return {3, 5, 7, g(7)};            // points 0,1,-1,2,inf: S = 1+2+4
        case 4: return {4, 7, 15, g(15)};          // 0,+-1,+-2,1/2,inf: S = 1+2+4+8
        case 8: {                                  // 0,+-1,...,+-64: S = sum 64^k, k<8
            uint64_t s = 0, p = 1;
            for (int k = 0; k < 8; ++k) { s += p; p *= 64; }
            return {8, 15, s, g(s)};
        }
        case 16: return {16, 31, tg_growthS_T16, g(tg_growthS_T16)};   // 31-point set (configs[4])
        // the paper's points 0, +-2^j (j < 31) at B = 32:
        // S = sum 2^(30 k) does not fit 64 bits; its limb count is generated
        case 32: return {32, 63, 0, tg_growthLimbs_P32};
        default: return {0, 0, 0, 0};
    }
}

// ------------------------------------------------------------------------
// accessors for the generated streaming programs
// ------------------------------------------------------------------------

// block k of a top-level (unsigned, row-major) operand row
struct InTop {
    const uint32_t* row;
    int b, lentop, B;
    __device__ __forceinline__ uint32_t load(int k, int t) const {
        const int len = (k == B - 1) ? lentop : b;
        return (t < len) ? __ldg(row + (size_t)k * b + t) : 0u;
    }
};

// block k of a signed interleaved parent operand (top block sign-extended)
struct InLevel {
    const uint32_t* col;
    size_t stride;
    int b, lentop, B;
    uint32_t fill;
    __device__ __forceinline__ uint32_t load(int k, int t) const {
        const int len = (k == B - 1) ? lentop : b;
        if (t < len) return __ldg(col + (size_t)(k * b + t) * stride);
        return (k == B - 1) ? fill : 0u;
    }
};

struct OutInterleaved {
    uint32_t* base;      // already offset by the instance column
    size_t stride_limb;  // distance between limbs of one value
    size_t stride_val;   // distance between consecutive values (points / coefficients)
    __device__ __forceinline__ void store(int j, int t, uint32_t x) const {
        base[(size_t)t * stride_limb + (size_t)j * stride_val] = x;
    }
};

// the 2B-1 child products of one parent: y_k limb t at (t*stride_limb + k*stride_val)
template <int NPTS>
struct InProducts {
    const uint32_t* base;
    size_t stride_limb, stride_val;
    int width;
    uint32_t fill[NPTS];
    __device__ __forceinline__ uint32_t load(int k, int t) const {
        return (t < width) ? __ldg(base + (size_t)t * stride_limb + (size_t)k * stride_val) : fill[k];
    }
};

// ------------------------------------------------------------------------
// point-set dispatch to the generated programs
// ------------------------------------------------------------------------
template <int B> struct PS;
template <> struct PS<3> {
    static constexpr int npts = 5;
    template <class I, class O> __device__ static void eval(const I& i, O& o, int n) { tg_eval_T3(i, o, n); }
    template <class I, class O> __device__ static void interp(const I& i, O& o, int n) { tg_interp_T3(i, o, n); }
};
template <> struct PS<4> {
    static constexpr int npts = 7;
    template <class I, class O> __device__ static void eval(const I& i, O& o, int n) { tg_eval_T4(i, o, n); }
    template <class I, class O> __device__ static void interp(const I& i, O& o, int n) { tg_interp_T4(i, o, n); }
};
template <> struct PS<8> {
    static constexpr int npts = 15;
    template <class I, class O> __device__ static void eval(const I& i, O& o, int n) { tg_eval_P8(i, o, n); }
    template <class I, class O> __device__ static void interp_even(const I& i, O& o, int n) { tg_interp_P8_even(i, o, n); }
    template <class I, class O> __device__ static void interp_odd(const I& i, O& o, int n) { tg_interp_P8_odd(i, o, n); }
};

// ------------------------------------------------------------------------
// step a2: evaluation.  One thread per (instance, operand).
//   TOP:   src = u or v row-major [count][n], unsigned
//   !TOP:  src = interleaved [n][count] two's complement
// out: interleaved [e][npts*count]; value of point k for instance c at column k*count + c
// ------------------------------------------------------------------------
template <int B, bool TOP>
__global__ void __launch_bounds__(128) k_eval(const uint32_t* __restrict__ srcU, const uint32_t* __restrict__ srcV,
                                              uint32_t* __restrict__ outU, uint32_t* __restrict__ outV,
                                              size_t count, int n, int b, int e) {
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= (srcV ? 2 : 1) * count) return;   // srcV = nullptr: one operand only
    const int which = gid >= count;
    const size_t c = which ? gid - count : gid;
    const uint32_t* src = which ? srcV : srcU;
    uint32_t* out = which ? outV : outU;
    const int lentop = n - (B - 1) * b;
    OutInterleaved o{out + c, (size_t)PS<B>::npts * count, count};
    if (TOP) {
        InTop in{src + c * (size_t)n, b, lentop, B};
        PS<B>::eval(in, o, e);
    } else {
        const uint32_t top = __ldg(src + (size_t)(n - 1) * count + c);
        InLevel in{src + c, count, b, lentop, B, (top >> 31) ? 0xFFFFFFFFu : 0u};
        PS<B>::eval(in, o, e);
    }
}

// ------------------------------------------------------------------------
// step a3: base case.  Register-resident product-scanning (Comba) schoolbook
// of two E-limb two's-complement operands; magnitudes multiplied with
// mad.lo.cc / madc.hi.cc / addc carry chains (-> IMAD.WIDE.U32 + IADD3.X),
// product sign applied while the columns are streamed out.
// ------------------------------------------------------------------------
#define TG_MADD(c0, c1, c2, a, b)                                    \
    asm volatile("mad.lo.cc.u32 %0, %3, %4, %0;\n\t"                 \
                 "madc.hi.cc.u32 %1, %3, %4, %1;\n\t"                \
                 "addc.u32 %2, %2, 0;"                               \
                 : "+r"(c0), "+r"(c1), "+r"(c2) : "r"(a), "r"(b))

template <int E>
__device__ __forceinline__ uint32_t load_abs(const uint32_t* __restrict__ src, size_t stride, uint32_t (&a)[E]) {
#pragma unroll
    for (int i = 0; i < E; ++i) a[i] = __ldg(src + (size_t)i * stride);
    const uint32_t neg = a[E - 1] >> 31;
    const uint32_t mask = 0u - neg;
    uint32_t carry = neg;
#pragma unroll
    for (int i = 0; i < E; ++i) {
        const uint32_t x = (a[i] ^ mask) + carry;
        carry = (x < carry) ? 1u : 0u;
        a[i] = x;
    }
    return neg;
}

template <int E>
__global__ void __launch_bounds__(128) k_base(const uint32_t* __restrict__ U, const uint32_t* __restrict__ V,
                                              uint32_t* __restrict__ P, size_t count) {
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    uint32_t a[E], b[E];
    const uint32_t sa = load_abs<E>(U + c, count, a);
    const uint32_t sb = load_abs<E>(V + c, count, b);
    const uint32_t neg = sa ^ sb;
    const uint32_t mask = 0u - neg;
    uint32_t ncarry = neg;
    uint32_t c0 = 0, c1 = 0, c2 = 0;
    uint32_t* out = P + c;
#pragma unroll
    for (int k = 0; k < 2 * E - 1; ++k) {
#pragma unroll
        for (int i = (k < E ? 0 : k - E + 1); i <= (k < E ? k : E - 1); ++i) {
            TG_MADD(c0, c1, c2, a[i], b[k - i]);
        }
        const uint32_t x = (c0 ^ mask) + ncarry;
        ncarry = (x < ncarry) ? 1u : 0u;
        out[(size_t)k * count] = x;
        c0 = c1;
        c1 = c2;
        c2 = 0;
    }
    out[(size_t)(2 * E - 1) * count] = (c0 ^ mask) + ncarry;
}

// generic base case for 40 < E <= 64 (operands staged in local memory)
__global__ void __launch_bounds__(128) k_base_generic(const uint32_t* __restrict__ U, const uint32_t* __restrict__ V,
                                                      uint32_t* __restrict__ P, size_t count, int E) {
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    uint32_t a[72], b[72];
    uint32_t sgn[2];
    for (int w = 0; w < 2; ++w) {
        const uint32_t* src = (w ? V : U) + c;
        uint32_t* d = w ? b : a;
        for (int i = 0; i < E; ++i) d[i] = __ldg(src + (size_t)i * count);
        const uint32_t neg = d[E - 1] >> 31, mask = 0u - neg;
        uint32_t carry = neg;
        for (int i = 0; i < E; ++i) {
            const uint32_t x = (d[i] ^ mask) + carry;
            carry = (x < carry) ? 1u : 0u;
            d[i] = x;
        }
        sgn[w] = neg;
    }
    const uint32_t neg = sgn[0] ^ sgn[1], mask = 0u - neg;
    uint32_t ncarry = neg, c0 = 0, c1 = 0, c2 = 0;
    for (int k = 0; k < 2 * E - 1; ++k) {
        const int lo = k < E ? 0 : k - E + 1, hi = k < E ? k : E - 1;
        for (int i = lo; i <= hi; ++i) TG_MADD(c0, c1, c2, a[i], b[k - i]);
        const uint32_t x = (c0 ^ mask) + ncarry;
        ncarry = (x < ncarry) ? 1u : 0u;
        P[(size_t)k * count + c] = x;
        c0 = c1; c1 = c2; c2 = 0;
    }
    P[(size_t)(2 * E - 1) * count + c] = (c0 ^ mask) + ncarry;
}

// ------------------------------------------------------------------------
// step a5: recomposition w = sum_j w_j 2^(32 b j) (Eq. 1.3) with carry
// propagation.  w_j are two's-complement streams of Lw limbs (sign-extended
// beyond); the sum is accumulated limb by limb with an unsigned 64-bit
// accumulator (at most 2B-1 terms per limb), which is exact for infinite
// two's-complement streams.
// ------------------------------------------------------------------------
template <int NPTS, bool TOP>
__device__ __forceinline__ void recompose(const uint32_t* __restrict__ W, size_t count, int Lw, int b,
                                          uint32_t* __restrict__ out, size_t out_stride, int wout) {
    // W: this instance's column: w_j limb t at W[(j*Lw + t)*count]; Lw = 2b+1.
    // Output limb P = s*b + r receives w_s[r], w_{s-1}[b+r], w_{s-2}[2b] (r = 0
    // only) and the sign fills of every w_j with j <= s-2 that has ended.
    uint32_t negfill[NPTS];
#pragma unroll
    for (int j = 0; j < NPTS; ++j) negfill[j] = W[((size_t)j * Lw + Lw - 1) * count] >> 31;
    const size_t sj = (size_t)Lw * count;
    uint64_t carry = 0;
    uint32_t lowfills = 0;   // number of negative w_j with j <= s-3
    const int nseg = (wout + b - 1) / b;
    for (int s = 0; s < nseg; ++s) {
        const bool hasA = s < NPTS, hasB = s >= 1 && s - 1 < NPTS, hasC = s >= 2 && s - 2 < NPTS;
        const uint32_t* pA = W + (size_t)(hasA ? s : 0) * sj;
        const uint32_t* pB = W + (size_t)(hasB ? s - 1 : 0) * sj + (size_t)b * count;
        uint32_t fillC = 0;
        if (hasC) {
#pragma unroll
            for (int j = 0; j < NPTS; ++j) if (j == s - 2) fillC = negfill[j];
        }
        const uint64_t lowconst = (uint64_t)lowfills * 0xFFFFFFFFull;
        const int rmax = min(b, wout - s * b);
        // r = 0: w_{s-2}[2b] is the last limb of w_{s-2}
        int r = 0;
        {
            uint64_t acc = carry + lowconst;
            if (hasA) acc += pA[0];
            if (hasB) acc += pB[0];
            if (hasC) acc += W[(size_t)(s - 2) * sj + (size_t)(2 * b) * count];
            out[(size_t)(s * b) * out_stride] = (uint32_t)acc;
            carry = acc >> 32;
            r = 1;
        }
        const uint64_t cconst = lowconst + (fillC ? 0xFFFFFFFFull : 0ull);
        for (; r + 4 <= rmax; r += 4) {
            uint32_t a[4], bb[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                a[q] = hasA ? pA[(size_t)(r + q) * count] : 0u;
                bb[q] = hasB ? pB[(size_t)(r + q) * count] : 0u;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint64_t acc = carry + cconst + a[q] + bb[q];
                out[(size_t)(s * b + r + q) * out_stride] = (uint32_t)acc;
                carry = acc >> 32;
            }
        }
        for (; r < rmax; ++r) {
            uint64_t acc = carry + cconst;
            if (hasA) acc += pA[(size_t)r * count];
            if (hasB) acc += pB[(size_t)r * count];
            out[(size_t)(s * b + r) * out_stride] = (uint32_t)acc;
            carry = acc >> 32;
        }
        if (hasC) lowfills += fillC;
    }
}

// ------------------------------------------------------------------------
// step a4 (+a5): interpolation of one parent per thread, then recomposition.
//   Pc:  child products, interleaved [2e][npts*count] (point k of parent c at column k*count + c)
//   W:   scratch [npts][Lw][count]
//   out: TOP ? row-major w[count][wout] : interleaved [wout][count]
// ------------------------------------------------------------------------
template <int B, bool TOP>
__global__ void __launch_bounds__(128) k_interp(const uint32_t* __restrict__ Pc, uint32_t* __restrict__ W,
                                                uint32_t* __restrict__ out, size_t count, int ywidth,
                                                int Lw, int b, int wout) {
    constexpr int NP = PS<B>::npts;
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    InProducts<NP> in;
    in.base = Pc + c;
    in.stride_limb = (size_t)NP * count;
    in.stride_val = count;
    in.width = ywidth;
#pragma unroll
    for (int k = 0; k < NP; ++k)
        in.fill[k] = (__ldg(in.base + (size_t)(ywidth - 1) * in.stride_limb + (size_t)k * count) >> 31) ? 0xFFFFFFFFu : 0u;
    OutInterleaved wo{W + c, count, (size_t)Lw * count};
    PS<B>::interp(in, wo, Lw);
    if (TOP) recompose<NP, true>(W + c, count, Lw, b, out + c * (size_t)wout, 1, wout);
    else recompose<NP, false>(W + c, count, Lw, b, out + c, count, wout);
}

// P8 (the paper's points, 15 values): the even and odd halves are independent
// and run on two adjacent lanes; the even lane recomposes.
template <bool TOP>
__global__ void __launch_bounds__(128) k_interp_p8(const uint32_t* __restrict__ Pc, uint32_t* __restrict__ W,
                                                   uint32_t* __restrict__ out, size_t count, int ywidth,
                                                   int Lw, int b, int wout) {
    constexpr int NP = 15;
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t c = gid >> 1;
    const int half = (int)(gid & 1);
    const bool active = c < count;
    if (active) {
        InProducts<NP> in;
        in.base = Pc + c;
        in.stride_limb = (size_t)NP * count;
        in.stride_val = count;
        in.width = ywidth;
#pragma unroll
        for (int k = 0; k < NP; ++k)
            in.fill[k] = (__ldg(in.base + (size_t)(ywidth - 1) * in.stride_limb + (size_t)k * count) >> 31) ? 0xFFFFFFFFu : 0u;
        OutInterleaved wo{W + c, count, (size_t)Lw * count};
        if (half == 0) PS<8>::interp_even(in, wo, Lw);
        else PS<8>::interp_odd(in, wo, Lw);
    }
    __syncwarp();
    if (active && half == 0) {
        if (TOP) recompose<NP, true>(W + c, count, Lw, b, out + c * (size_t)wout, 1, wout);
        else recompose<NP, false>(W + c, count, Lw, b, out + c, count, wout);
    }
}

}  // namespace tg
#include "fused_bottom.cuh"
#include "fused_dc.cuh"
#include "longvec.cuh"
#include "longvec2.cuh"
#include "level34.cuh"
#include "ntt.cuh"
#include "lazy.cuh"
#include "toplevel.cuh"
#include "toplevel_cls.cuh"
#include "tc_base.cuh"
namespace tg {

// ------------------------------------------------------------------------
// planner (step a6): the recursion shape and the workspace layout
// ------------------------------------------------------------------------
struct Level {
    int B = 0;          // 0 = base case
    size_t count = 0;   // instances at this level
    int n = 0;          // operand width in limbs (unsigned at level 0, signed below)
    int b = 0, lentop = 0;
    int e = 0;          // child operand width
    int Lw = 0;         // interpolation output width per coefficient
    int npts = 0;
    bool lng = false;   // long-vector (limb-parallel) level: row-major child layouts
    bool res = false;   // ... run instance-resident (one CTA per instance, level34.cuh)
    bool lazy = false;  // ... run lazy (csrc/lazy.cuh): carry-save values, deferred division
    int Wy = 0, Wx = 0; // lazy: positions of the child products read / of the product written
    size_t offU = 0, offV = 0, offP = 0, offW = 0;   // child operands/products, this level's scratch
    size_t offLzU = 0, offLzV = 0, offLzP = 0;        // lazy children (LO | HI) and lazy child products
};

struct Plan {
    std::vector<Level> lv;   // lv[0..L-1] Toom levels, lv[L] = base level
    size_t bytes = 0;
    bool fused = false;      // bottom Toom level runs as k_fused_bottom
    bool signed_in = false;  // user operands are two's complement (stage export)
    bool square = false;     // v = u: V children alias U children, squaring base case
    // long-vector levels: slot pool, scan status, tile counters, op descriptors
    size_t offSlots = 0, offStatus = 0, offCtr = 0, offDesc = 0;
    size_t nStatus = 0, nCtr = 0, nDesc = 0;
    // boundary long level (its children feed an instance-parallel level):
    // row-major staging of its children / their products, transposed to and
    // from the interleaved layout of the level below
    int bnd = -1;
    size_t offT = 0;
    size_t offEDesc = 0;     // multi-output evaluation descriptors
    size_t offBDesc = 0;     // wide-multiplier multi-output descriptors (matrix-form T16)
    bool top_warp = false;   // top interpolation one warp per product (fused level writes row-major)
    int c2mode = 0;          // C2 shape: 1 top level by classes (toplevel_cls.cuh), 2 + deferred bottom (fused_dc.cuh)
    bool lzdc = false;       // T3 bottom under the lazy block: X = 6 y, the factor joins the finishing division
    // lazy block [lz0, lz1) of long levels (csrc/lazy.cuh): the product of
    // their common denominators 2^lz_s lz_o, the top lazy output X and the
    // two-pass tile records of the finishing scans
    int lz0 = -1, lz1 = -1;
    std::vector<uint32_t> lz_o;   // odd part of prod Dc as word factors (one finishing division each)
    int lz_s = 0;
    size_t offLzX = 0, offLzT = 0, offLzTiles = 0, nLzTiles = 0;
};

// generated long-vector tables of a point set
struct LongTables {
    const tg_lterm* et; const tg_lop* eo; int neo;
    const tg_lterm* it; const tg_lop* io; const int* iout; int nio; int nslots; int lag;
};
static bool long_tables(int B, LongTables& T) {
#define TG_LT(NM)                                                                                      \
    T = {tg_lt_##NM##_eval, tg_lo_##NM##_eval, tg_lnops_##NM##_eval, tg_lt_##NM##_interp,              \
         tg_lo_##NM##_interp, tg_lout_##NM##_interp, tg_lnops_##NM##_interp, tg_lnslots_##NM##_interp,  \
         tg_llag_##NM##_interp};                                                                       \
    return true;
    switch (B) {
        case 3: TG_LT(T3)
        case 4: TG_LT(T4)
        case 8: TG_LT(P8)
        case 16: TG_LT(T16)
        case 32: TG_LT(P32)
        default: return false;
    }
#undef TG_LT
}
static int long_Wt(const Level& L) {
    LongTables T;
    long_tables(L.B, T);
    return L.Lw + T.lag;
}
static size_t long_tiles(size_t count, int W) { return count * (size_t)((W + 32 * 4 - 1) / (32 * 4)); }

// base widths with a fused bottom-level instantiation (C1 33, C2 18, C3/C4/C5 23, ...)
static bool fused_E_supported(int E) {
    return E == 6 || E == 9 || E == 18 || E == 23 || E == 27 || E == 33;
}
static bool g_disable_fused = false;

static bool split_ok(int n, int B) {
    const int b = (n + B - 1) / B;
    return n >= 2 * B && n - (B - 1) * b >= 1;   // top block must be non-empty
}

// B of the level at `depth` for an n-limb operand (0 = schoolbook base case).
// A requested top-level B that cannot split n (top block empty) falls back to
// the lower levels' size rule.
static int choose_B(const toom_plan_t& p, int depth, int n) {
    if (depth == 0 && p.top_B && split_ok(n, p.top_B)) return p.top_B;
    int B;
    if ((size_t)n > p.t4) B = 4;
    else if ((size_t)n > p.t3) B = 3;
    else return 0;
    if (!split_ok(n, B)) return (B == 4 && split_ok(n, 3)) ? 3 : 0;
    return B;
}

static const bool g_eval_v4 = [] {      // TOOM_EVAL_V4=0: k_eval_top_rows only
    const char* e = getenv("TOOM_EVAL_V4");
    return e ? atoi(e) != 0 : true;
}();
static const bool g_its_static = [] {   // TOOM_ITS_STATIC=0: generic shapes only (top interpolation, fused bottom)
    const char* e = getenv("TOOM_ITS_STATIC");
    return e ? atoi(e) != 0 : true;
}();
static int g_top_stream = 2;   // 3: one warp per product, 2: smem kernel, 1: one-pass stream, 0: per-row kernel
// default long-vector rule: levels whose operands exceed this many limbs
static int g_long_min_n = [] {
    const char* e = getenv("TOOM_LONG_MIN_N");
    return e ? atoi(e) : 2048;
}();
// ... and fewer than this many instances (many instances: one thread per
// instance has parallelism enough, the per-tile scans of the long kernels cost more)
static int g_long_max_count = [] {
    const char* e = getenv("TOOM_LONG_MAX_COUNT");
    return e ? atoi(e) : 8000;   // C5: 220 -> 150 ms (levels 4, 5 instance-parallel); C4 unchanged
}();

// instance-resident levels (level34.cuh): operands of at most this many limbs
static int g_res_max_n = [] {
    const char* e = getenv("TOOM_RES_MAX_N");
    return e ? atoi(e) : 4200;
}();
// ... and at least this many (below: one thread per instance has parallelism
// enough and no scan overhead; measured on C4's 1026- and 258-limb levels)
static int g_res_min_n = [] {
    const char* e = getenv("TOOM_RES_MIN_N");
    return e ? atoi(e) : 2000;
}();
static bool g_res_on = [] {
    const char* e = getenv("TOOM_RES");
    return e ? atoi(e) != 0 : true;
}();

// lazy long levels (csrc/lazy.cuh); TOOM_LAZY=0 runs them on the two-pass
// long-op executor instead (tests compare both)
static int g_lazy = [] {
    const char* e = getenv("TOOM_LAZY");
    return e ? atoi(e) : 1;
}();

// the matrix-form Toom-16 interpolation (f1) instead of the 459-op staged
// Newton program: TOOM_T16_MATRIX=0 restores the latter (tests compare both)
static bool g_t16_matrix = [] {
    const char* e = getenv("TOOM_T16_MATRIX");
    return e ? atoi(e) != 0 : true;
}();
// C2-shaped batches: the top level as one division over the common
// denominator (csrc/toplevel_cls.cuh) and the bottom level with that
// denominator deferred to it (csrc/fused_dc.cuh); TOOM_C2_CLS=0 /
// TOOM_DEFERRED_BOTTOM=0 run the per-row kernels instead (tests compare all)
// the Toom-3 bottom under the lazy levels (C4, C5) with its denominator 6
// deferred into the lazy block's finishing division (csrc/fused_dc.cuh);
// TOOM_LAZY_BOTTOM_DC=0 runs the per-row fused kernel instead
static bool g_lzdc = [] {
    const char* e = getenv("TOOM_LAZY_BOTTOM_DC");
    return e ? atoi(e) != 0 : true;
}();
static int g_c2mode = [] {
    const char* a = getenv("TOOM_C2_CLS");
    const char* b = getenv("TOOM_DEFERRED_BOTTOM");
    const bool cls = a ? atoi(a) != 0 : true;
    const bool dc = b ? atoi(b) != 0 : true;
    return cls ? (dc ? 2 : 1) : 0;
}();
constexpr int F1_SLOTS = 61;   // E, O, R, T (15 each) + y'
static int long_nslots(int B, int nslots) { return (B == 16 && g_t16_matrix) ? std::max(nslots, F1_SLOTS) : nslots; }

// one warp per product (k_interp_top_warp) needs the products row-major; CH
// positions per lane, CH = ceil((2n+1)/32) rounded up to an instantiated size
static int top_warp_ch(const Level& Lv) {
    const int need = (2 * Lv.n + 1 + 31) / 32;
    if (Lv.B != 3 && Lv.B != 4) return 0;
    for (int c : {9, 17, 33})
        if (need <= c) return c;
    return 0;
}

static toom_status make_plan(int n, size_t batch, const toom_plan_t& p, Plan& plan, bool top_long = false,
                             bool square = false) {
    plan.square = square;
    plan.lv.clear();
    size_t count = batch;
    int width = n;
    for (int depth = 0;; ++depth) {
        Level L;
        L.count = count;
        L.n = width;
        L.B = choose_B(p, depth, width);
        if (L.B == 0) {
            if (width > 64) return TOOM_EUNSUPPORTED;
            plan.lv.push_back(L);
            break;
        }
        const PSDesc d = ps_desc(L.B);
        if (!d.B) return TOOM_EINVAL;
        L.npts = d.npts;
        L.b = (width + L.B - 1) / L.B;
        L.lentop = width - (L.B - 1) * L.b;
        L.e = L.b + d.grow;
        L.Lw = 2 * L.b + 1;
        plan.lv.push_back(L);
        count *= (size_t)d.npts;
        width = L.e;
        if (depth > 40) return TOOM_EUNSUPPORTED;
    }
    // long-vector levels: a prefix of the Toom levels with few instances
    {
        // default (long_count = 0): operands longer than 2048 limbs (few,
        // long vectors: one thread per instance would stream too long);
        // long_count = 1: never; otherwise: levels with < long_count instances
        // Default plans also run the levels below a long level (and a top
        // level of few instances) with operands of at most g_res_max_n limbs
        // instance-resident (level34.cuh) down to the fused bottom level, so
        // that the whole recursion keeps row-major layouts.
        LongTables T;
        const size_t NL = plan.lv.size() - 1;   // Toom levels
        const Level& Bt = plan.lv[NL - (NL ? 1 : 0)];
        const bool fusable = NL >= 1 && !g_disable_fused && (Bt.B == 3 || Bt.B == 4) && fused_E_supported(Bt.e) &&
                             Bt.e == Bt.b + 1 && Bt.Lw == 2 * Bt.b + 1 && 2 * Bt.e > Bt.Lw &&
                             2 * Bt.n <= (2 * Bt.B - 1) * 2 * Bt.e;
        for (size_t l = 0; l < NL; ++l) {
            Level& L = plan.lv[l];
            const bool want = L.B == 16 || L.B == 32 || (top_long && l == 0) ||   // T16/P32: no instance-parallel program
                              (p.long_count == 0 ? (L.n > g_long_min_n && L.count < (size_t)g_long_max_count)
                                                 : (p.long_count > 1 && L.count < p.long_count)) ||
                              // below a long level, operands too long to be resident stay long
                              (p.long_count == 0 && g_res_on && l > 0 && plan.lv[l - 1].lng && L.n > g_res_max_n &&
                               L.count < (size_t)g_long_max_count);
            const bool resok = p.long_count == 0 && g_res_on && (L.B == 3 || L.B == 4) && L.n <= g_res_max_n &&
                               L.n >= g_res_min_n &&
                               l + 1 < NL && L.count < (size_t)g_long_max_count &&   // many instances: one thread each (C5: 125 vs 158 ms)
                               res_interp_smem(L.B, 2 * L.e, L.Lw, res_threads(L.Lw + 1)) <= 200 * 1024;
            if (resok && (l > 0 || want)) { L.lng = true; L.res = true; }
            else if (want && long_tables(L.B, T)) L.lng = true;
            else if (l > 0 && plan.lv[l - 1].lng && resok) { L.lng = true; L.res = true; }
            else break;
        }

        for (size_t l = 0; l + 1 < plan.lv.size(); ++l)
            if ((plan.lv[l].B == 16 || plan.lv[l].B == 32) && !plan.lv[l].lng) return TOOM_EUNSUPPORTED;   // long only
    }
    // lazy block (csrc/lazy.cuh): from the first long Toom-3/4 level (below a
    // long Toom-16/P32 top, or at the top) down to the level above the fused
    // bottom level (every level in between is elementwise when lazy, however
    // many instances it has); without a fused bottom level, the long,
    // non-resident prefix only.  The odd part of prod Dc is kept as word
    // factors for the finishing divisions.
    plan.lz0 = plan.lz1 = -1;
    plan.lz_o.clear();
    plan.lz_s = 0;
    if (g_lazy) {
        const size_t NL = plan.lv.size() - 1;
        const Level& Bt = plan.lv[NL - (NL ? 1 : 0)];
        const bool fusable = NL >= 2 && !g_disable_fused && (Bt.B == 3 || Bt.B == 4) && fused_E_supported(Bt.e) &&
                             Bt.e == Bt.b + 1 && Bt.Lw == 2 * Bt.b + 1 && 2 * Bt.e > Bt.Lw &&
                             2 * Bt.n <= (2 * Bt.B - 1) * 2 * Bt.e;
        const size_t fl = fusable ? NL - 1 : NL;   // first level that stays non-lazy
        uint64_t word = 1;
        for (size_t l = 0; l < fl; ++l) {
            Level& L = plan.lv[l];
            const bool t34 = (L.B == 3 || L.B == 4) && L.e == L.b + 1 && l + 1 < NL;
            const bool ok = t34 && (plan.lz0 >= 0 ? (fusable || (L.lng && !L.res)) : (L.lng && (fusable || !L.res)));
            if (!ok) {
                if (plan.lz0 >= 0 || !L.lng) break;
                continue;
            }
            const uint64_t o = L.B == 3 ? tg_combO_T3 : tg_combO_T4;
            const int sh = L.B == 3 ? tg_combS_T3 : tg_combS_T4;
            if (plan.lz_s + sh > 32 * (LV_MAXHALO - 2)) break;
            if (plan.lz0 < 0) plan.lz0 = (int)l;
            plan.lz1 = (int)l + 1;
            if (word * o > 0xFFFFFFFFull) { plan.lz_o.push_back((uint32_t)word); word = 1; }
            word *= o;
            plan.lz_s += sh;
            L.lazy = true;
            L.lng = true;
            L.res = false;
        }
        if (word > 1) plan.lz_o.push_back((uint32_t)word);
        if (plan.lz0 >= 0) {
            // product widths, deepest first: normalised 2e below the block
            for (int l = plan.lz1 - 1; l >= plan.lz0; --l) {
                Level& L = plan.lv[l];
                L.Wy = (l == plan.lz1 - 1) ? 2 * L.e : plan.lv[l + 1].Wx;
                L.Wx = (2 * L.B - 2) * L.b + L.Wy + 1;
                if ((L.Wy + L.b - 1) / L.b > 4) return TOOM_EUNSUPPORTED;
            }
            // levels below the block are not long any more
            for (size_t l = plan.lz1; l < NL; ++l) { plan.lv[l].lng = false; plan.lv[l].res = false; }
        }
    }
    // fused bottom level?
    plan.fused = false;
    if (plan.lv.size() >= 2 && !g_disable_fused && !plan.lv[plan.lv.size() - 2].lng) {
        const Level& Bt = plan.lv[plan.lv.size() - 2];
        if ((Bt.B == 3 || Bt.B == 4) && fused_E_supported(Bt.e) && Bt.e == Bt.b + 1 && Bt.Lw == 2 * Bt.b + 1 && 2 * Bt.e > Bt.Lw &&
            2 * Bt.n <= (2 * Bt.B - 1) * 2 * Bt.e)
            plan.fused = true;
    }
    // the Toom-3 bottom of 66-limb parents right under the lazy block: its
    // common denominator 6 = 2 * 3 joins the block's finishing division
    plan.lzdc = false;
    if (g_lzdc && g_its_static && plan.fused && !square && plan.lz1 >= 1 &&
        (size_t)plan.lz1 + 2 == plan.lv.size()) {
        const Level& Bt = plan.lv[plan.lz1];
        if (Bt.B == 3 && Bt.n == 66 && Bt.b == 22 && Bt.e == 23 && Bt.Lw == 45 &&
            plan.lz_s + tg_combS_T3 <= 32 * (LV_MAXHALO - 2)) {
            plan.lzdc = true;
            if (!plan.lz_o.empty() && (uint64_t)plan.lz_o.back() * tg_combO_T3 <= 0xFFFFFFFFull)
                plan.lz_o.back() *= tg_combO_T3;
            else
                plan.lz_o.push_back(tg_combO_T3);
            plan.lz_s += tg_combS_T3;
        }
    }
    // a batched top level directly above the fused level: its interpolation
    // can run one warp per product on row-major products (fused MODE 3)
    plan.top_warp = plan.fused && plan.lv.size() == 3 && !plan.lv[0].lng && g_top_stream == 3 &&
                    top_warp_ch(plan.lv[0]) > 0 && plan.lv[0].Lw == 2 * plan.lv[0].b + 1;
    // the C2 shape (256 -> 65 -> 18 limbs, Toom-4 twice, batched)
    const bool c2shape = plan.fused && !square && plan.lv.size() == 3 && !plan.lv[0].lng && !plan.top_warp &&
                         plan.lv[0].B == 4 && plan.lv[0].n == 256 && plan.lv[0].b == 64 && plan.lv[0].e == 65 &&
                         plan.lv[0].Lw == 129 && plan.lv[1].B == 4 && plan.lv[1].n == 65 && plan.lv[1].b == 17 &&
                         plan.lv[1].e == 18 && plan.lv[1].Lw == 35;
    plan.c2mode = (c2shape && g_its_static && g_top_stream == 2) ? g_c2mode : 0;
    // workspace layout
    size_t off = 0;
    auto take = [&](size_t limbs) { size_t o = off; off += ((limbs * 4 + 255) / 256) * 256; return o; };
    const size_t nstaged = plan.lv.size() - 1 - (plan.fused ? 1 : 0);
    for (size_t l = 0; l < nstaged; ++l) {
        Level& L = plan.lv[l];
        const size_t cc = L.count * (size_t)L.npts;
        if (L.lazy) {
            // lazy children (LO | HI) and, above the deepest lazy level, the
            // lazy child products in the same region (the children are dead
            // once the level below has evaluated them)
            const bool deepest = (int)l + 1 == plan.lz1;
            const bool deep_il = (size_t)plan.lz1 + 1 >= plan.lv.size() || !plan.lv[plan.lz1].lng;
            const size_t ch = (deepest && deep_il) ? 0 : (size_t)(square ? 2 : 4) * L.e * cc;
            const size_t pr = deepest ? 0 : (size_t)2 * plan.lv[l + 1].Wx * cc;
            const size_t reg = take(std::max(ch, pr));
            L.offLzU = reg;
            L.offLzV = square ? reg : reg + (size_t)2 * L.e * cc * 4;
            L.offLzP = reg;
            if (!deepest) continue;   // no normalised children / products
        }
        L.offU = take((size_t)L.e * cc);
        L.offV = square ? L.offU : take((size_t)L.e * cc);   // squaring: V = U
        L.offP = take((size_t)2 * L.e * cc);
        L.offW = L.lng ? 0 : take((size_t)L.npts * L.Lw * L.count);
    }
    if (plan.lz0 >= 0) {
        const Level& L0 = plan.lv[plan.lz0];
        const Level& Ld = plan.lv[plan.lz1 - 1];
        plan.offLzX = take((size_t)2 * L0.Wx * L0.count);
        if (plan.lz_o.size() > 1) plan.offLzT = take((size_t)2 * L0.Wx * L0.count);   // two normalised intermediates
        plan.nLzTiles = std::max((size_t)L0.count * (size_t)((L0.Wx + LV_TL - 1) / LV_TL),
                                 (size_t)Ld.count * Ld.npts * (size_t)((Ld.e + LV_TL - 1) / LV_TL));
        plan.offLzTiles = take((plan.nLzTiles * sizeof(LTile) + 3) / 4);
    }
    size_t slot_limbs = 0, tiles = 0, nops = 0;
    for (size_t l = 0; l < nstaged; ++l) {
        const Level& L = plan.lv[l];
        if (!L.lng || L.res || L.lazy) continue;
        LongTables T;
        long_tables(L.B, T);
        const int Wt = long_Wt(L);
        slot_limbs = std::max(slot_limbs, (size_t)long_nslots(L.B, T.nslots) * L.count * Wt);
        tiles = std::max(tiles, long_tiles(L.count, std::max(std::max(Wt, L.e), 2 * L.n)));
        tiles = std::max(tiles, long_tiles(L.count, std::max(L.e, L.Lw)) * (size_t)L.npts);   // multi-output ops
        nops += 2 * (size_t)T.neo + T.nio + 1 + 2;
    }
    {
        size_t Tl = 0;
        while (Tl + 1 < plan.lv.size() && plan.lv[Tl].lng) ++Tl;
        const size_t nTL = plan.lv.size() - 1;
        if (Tl >= 1 && Tl < nstaged && !plan.lv[Tl - 1].lazy) {   // level Tl is a staged instance-parallel Toom level
            const Level& L = plan.lv[Tl - 1];
            plan.bnd = (int)(Tl - 1);
            plan.offT = take((size_t)2 * L.e * L.count * L.npts);
        }
        (void)nTL;
    }
    if (nops) {
        plan.offSlots = take(slot_limbs);
        plan.nStatus = tiles;
        plan.offStatus = take((tiles * sizeof(LStatus) + 3) / 4);
        plan.nCtr = nops;
        plan.offCtr = take(nops);
        plan.nDesc = nops;
        plan.offDesc = take((nops * sizeof(LOpDev) + 3) / 4);
        plan.offEDesc = take((nops * sizeof(LMultiDev) + 3) / 4);
        plan.offBDesc = take((nops * sizeof(LBigDev) + 3) / 4);
    }
    plan.bytes = off;
    return TOOM_OK;
}

// ------------------------------------------------------------------------
// workspace + error state
// ------------------------------------------------------------------------
// Workspace.  Library-owned buffers are kept PER STREAM (calls on different
// streams never share scratch memory; a buffer grows only after its own
// stream has drained).  A caller-provided buffer (toom_set_workspace) is
// shared by every stream: a call holds it from the first use to the end of
// its enqueue and records an event; a call on another stream first waits for
// that event (stream-ordered, no host sync).
static std::mutex g_ws_mu;
struct WsEntry { cudaStream_t st; void* p; size_t bytes; };
static std::vector<WsEntry> g_ws_list;   // library-owned, one per stream
static void* g_user_ws = nullptr;        // caller-owned (toom_set_workspace)
static size_t g_user_bytes = 0;
static std::mutex g_user_mu;             // held by the call using g_user_ws
static cudaEvent_t g_user_ev = nullptr;
static cudaStream_t g_user_last = nullptr;
static bool g_user_used = false;
static thread_local toom_status t_last = TOOM_OK;
static thread_local size_t t_launches = 0;

// ---- optional per-launch CUDA-event profiling (bench.py roofline) ----
enum { CAT_EVAL = 0, CAT_BASE = 1, CAT_INTERP = 2, CAT_OTHER = 3, NCAT = 4 };
struct ProfRec { int cat; cudaEvent_t a, b; };
static thread_local bool t_prof = false;
static thread_local std::vector<ProfRec> t_prof_recs;
static thread_local std::vector<cudaEvent_t> t_prof_pool;
static thread_local cudaStream_t t_prof_stream = nullptr;
static cudaEvent_t prof_event() {
    if (!t_prof_pool.empty()) { cudaEvent_t e = t_prof_pool.back(); t_prof_pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
struct ProfScope {
    bool on; ProfRec r;
    ProfScope(int cat, cudaStream_t st) : on(t_prof) {
        if (on) { r.cat = cat; r.a = prof_event(); r.b = prof_event(); cudaEventRecord(r.a, st); t_prof_stream = st; }
    }
    void done(cudaStream_t st) { if (on) { cudaEventRecord(r.b, st); t_prof_recs.push_back(r); on = false; } }
};

static toom_status fail(toom_status s) {
    if (s != TOOM_OK) t_last = s;
    return s;
}

// a per-call workspace (the pipelined host entry point runs several chunks
// concurrently, each with its own workspace)
static thread_local void* t_ws_override = nullptr;
static thread_local size_t t_ws_override_bytes = 0;

// A workspace lease: ws_acquire(bytes, stream) gives the scratch for one call
// on `stream`; ws_release() ends it (records the caller-buffer event).
struct WsLease {
    bool user = false;
    cudaStream_t st = nullptr;
};
static thread_local WsLease t_lease;
static thread_local int t_lease_depth = 0;

static toom_status get_ws(size_t bytes, void** out, cudaStream_t st) {
    if (t_ws_override) {
        if (bytes > t_ws_override_bytes) return TOOM_ENOMEM;
        *out = t_ws_override;
        return TOOM_OK;
    }
    if (t_lease_depth > 0) return TOOM_EINVAL;   // one lease per call
    {
        std::lock_guard<std::mutex> g(g_ws_mu);
        if (!g_user_ws) {
            for (auto& e : g_ws_list) {
                if (e.st != st) continue;
                if (bytes <= e.bytes) { *out = e.p; ++t_lease_depth; t_lease = WsLease{false, st}; return TOOM_OK; }
                // grow: only this stream uses the buffer, so draining it suffices
                cudaStreamSynchronize(st);
                cudaFree(e.p);
                e.p = nullptr;
                e.bytes = 0;
                if (cudaMalloc(&e.p, bytes) != cudaSuccess) { cudaGetLastError(); return TOOM_ENOMEM; }
                e.bytes = bytes;
                *out = e.p;
                ++t_lease_depth;
                t_lease = WsLease{false, st};
                return TOOM_OK;
            }
            WsEntry e{st, nullptr, 0};
            if (cudaMalloc(&e.p, bytes) != cudaSuccess) { cudaGetLastError(); return TOOM_ENOMEM; }
            e.bytes = bytes;
            g_ws_list.push_back(e);
            *out = e.p;
            ++t_lease_depth;
            t_lease = WsLease{false, st};
            return TOOM_OK;
        }
    }
    // caller-owned buffer: exclusive until ws_release
    g_user_mu.lock();
    if (!g_user_ws || bytes > g_user_bytes) { g_user_mu.unlock(); return TOOM_ENOMEM; }
    if (!g_user_ev) cudaEventCreateWithFlags(&g_user_ev, cudaEventDisableTiming);
    if (g_user_used && g_user_last != st) cudaStreamWaitEvent(st, g_user_ev, 0);
    *out = g_user_ws;
    ++t_lease_depth;
    t_lease = WsLease{true, st};
    return TOOM_OK;
}

static void ws_release() {
    if (t_lease_depth == 0) return;
    --t_lease_depth;
    if (t_lease.user) {
        cudaEventRecord(g_user_ev, t_lease.st);
        g_user_last = t_lease.st;
        g_user_used = true;
        g_user_mu.unlock();
    }
    t_lease = WsLease{};
}
struct WsGuard {
    bool on = false;
    ~WsGuard() { if (on) ws_release(); }
};

static inline unsigned nblk(size_t threads, int bs = 128) { return (unsigned)((threads + bs - 1) / bs); }

static bool g_eval_p8 = [] {   // TOOM_EVAL_P8=0: the per-product streaming program for C3's top level
    const char* e = getenv("TOOM_EVAL_P8");
    return e ? atoi(e) != 0 : true;
}();
static toom_status launch_eval(int B, bool top, const uint32_t* su, const uint32_t* sv, uint32_t* ou, uint32_t* ov,
                               size_t count, int n, int b, int e, cudaStream_t st) {
    const unsigned g = nblk((sv ? 2 : 1) * count);
    if (g == 0) return TOOM_OK;
    ProfScope ps(CAT_EVAL, st);
    if (B == 8 && top && sv && g_eval_p8) {   // the paper's points: pairs of +-2^i by funnel shifts
        k_eval_top_p8<<<(unsigned)((count + 7) / 8), 128, 0, st>>>(su, sv, ou, ov, count, n, b, e);
        ps.done(st);
        ++t_launches;
        return TOOM_OK;
    }
#define TG_EV(BB)                                                                          \
    if (top) k_eval<BB, true><<<g, 128, 0, st>>>(su, sv, ou, ov, count, n, b, e);          \
    else k_eval<BB, false><<<g, 128, 0, st>>>(su, sv, ou, ov, count, n, b, e);
    switch (B) {
        case 3: TG_EV(3); break;
        case 4: TG_EV(4); break;
        case 8: TG_EV(8); break;
        default: return TOOM_EINVAL;
    }
#undef TG_EV
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

// few instances (few threads for the per-thread programs) but long rows: the
// row-parallel interpolation has 2B-3 times the threads (C5 level 4)
static int g_rows_max_count = [] {
    const char* e = getenv("TOOM_ROWS_MAX_COUNT");
    return e ? atoi(e) : 24000;   // C4's 16807-instance level: 4.59 -> 4.29 ms of interpolation
}();

static bool g_p8_rows_split = [] {   // TOOM_P8_ROWS_SPLIT=0: the generic-multiplier row kernel (A/B timing)
    const char* e = getenv("TOOM_P8_ROWS_SPLIT");
    return e ? atoi(e) != 0 : true;
}();
static toom_status launch_interp(int B, bool top, const uint32_t* Pc, uint32_t* W, uint32_t* out, size_t count,
                                 int ywidth, int Lw, int b, int wout, cudaStream_t st) {
    if (count == 0) return TOOM_OK;
    ProfScope ps(CAT_INTERP, st);
    switch (B) {
        case 3:
        case 4:
            // batched Toom-3/4 levels: row-parallel interpolation + segment
            // recomposition only in top-interpolation mode 4 (measured slower
            // than the per-thread programs at C2-C5's shapes: every row re-reads
            // all 2B-1 products)
            if ((g_top_stream == 4 || (g_top_stream != 0 && count < (size_t)g_rows_max_count)) && Lw == 2 * b + 1 && (size_t)Lw >= 3 * (size_t)((wout + b - 1) / b) && ywidth > Lw) {
                // rows in parallel (one thread per interior row and product) +
                // segment-parallel recomposition; W row 0 holds the segment carries
                const int nseg = (wout + b - 1) / b, NP = 2 * B - 1;
                if (B == 3) k_interp_rows_w<3><<<nblk((size_t)(NP - 2) * count), 128, 0, st>>>(Pc, W, count, ywidth, Lw);
                else k_interp_rows_w<4><<<nblk((size_t)(NP - 2) * count), 128, 0, st>>>(Pc, W, count, ywidth, Lw);
                RecompArgs A{Pc, W, out, top ? (long long)wout : 1, top ? 1 : (long long)count, W, count, NP, Lw, b, wout,
                             nseg, 1};
                k_recomp_seg<<<nblk((size_t)nseg * count), 128, 0, st>>>(A);
                k_recomp_fix<<<nblk(count), 128, 0, st>>>(W, count, nseg);
                k_recomp_apply<<<nblk((size_t)nseg * count), 128, 0, st>>>(A);
                t_launches += 3;
                break;
            }
            if (B == 4) {
                if (top) k_interp<4, true><<<nblk(count), 128, 0, st>>>(Pc, W, out, count, ywidth, Lw, b, wout);
                else k_interp<4, false><<<nblk(count), 128, 0, st>>>(Pc, W, out, count, ywidth, Lw, b, wout);
                break;
            }
            if (top) k_interp<3, true><<<nblk(count), 128, 0, st>>>(Pc, W, out, count, ywidth, Lw, b, wout);
            else k_interp<3, false><<<nblk(count), 128, 0, st>>>(Pc, W, out, count, ywidth, Lw, b, wout);
            break;
        case 8:
            // (top-interpolation mode 0 keeps the one-lane-per-half-program kernel)
            if (top && g_top_stream != 0 && Lw == 2 * b + 1 && (size_t)Lw >= 3 * (size_t)((wout + b - 1) / b)) {
                // rows in parallel (one thread per row and product), then the
                // segment-parallel recomposition (row 0's scratch holds the carries)
                const int nseg = (wout + b - 1) / b;
                if (g_p8_rows_split) k_interp_rows_p8s<<<(unsigned)(14 * ((count + 127) / 128)), 128, 0, st>>>(Pc, W, count, ywidth, Lw);
                else k_interp_rows_p8<<<nblk(14 * count), 128, 0, st>>>(Pc, W, count, ywidth, Lw);
                RecompArgs A{Pc, W, out, (long long)wout, 1, W, count, 15, Lw, b, wout, nseg, 0};
                k_recomp_seg<<<nblk((size_t)nseg * count), 128, 0, st>>>(A);
                k_recomp_fix<<<nblk(count), 128, 0, st>>>(W, count, nseg);
                k_recomp_apply<<<nblk((size_t)nseg * count), 128, 0, st>>>(A);
                t_launches += 3;
                break;
            }
            if (top) k_interp_p8<true><<<nblk(2 * count), 128, 0, st>>>(Pc, W, out, count, ywidth, Lw, b, wout);
            else k_interp_p8<false><<<nblk(2 * count), 128, 0, st>>>(Pc, W, out, count, ywidth, Lw, b, wout);
            break;
        default: return TOOM_EINVAL;
    }
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

template <int E>
static void launch_base_E(const uint32_t* U, const uint32_t* V, uint32_t* P, size_t count, cudaStream_t st) {
    k_base<E><<<nblk(count), 128, 0, st>>>(U, V, P, count);
}

static toom_status launch_base(int E, const uint32_t* U, const uint32_t* V, uint32_t* P, size_t count, cudaStream_t st) {
    if (count == 0) return TOOM_OK;
    ProfScope ps(CAT_BASE, st);
    switch (E) {
#define TG_BC(k) case k: launch_base_E<k>(U, V, P, count, st); break;
        TG_BC(1) TG_BC(2) TG_BC(3) TG_BC(4) TG_BC(5) TG_BC(6) TG_BC(7) TG_BC(8)
        TG_BC(9) TG_BC(10) TG_BC(11) TG_BC(12) TG_BC(13) TG_BC(14) TG_BC(15) TG_BC(16)
        TG_BC(17) TG_BC(18) TG_BC(19) TG_BC(20) TG_BC(21) TG_BC(22) TG_BC(23) TG_BC(24)
        TG_BC(25) TG_BC(26) TG_BC(27) TG_BC(28) TG_BC(29) TG_BC(30) TG_BC(31) TG_BC(32)
        TG_BC(33) TG_BC(34) TG_BC(35) TG_BC(36) TG_BC(37) TG_BC(38) TG_BC(39) TG_BC(40)
#undef TG_BC
        default:
            if (E < 1 || E > 72) return TOOM_EINVAL;
            k_base_generic<<<nblk(count), 128, 0, st>>>(U, V, P, count, E);
    }
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

template <int B, int E, int TOP>
static void launch_fused_t(const Level& Lv, const uint32_t* su, const uint32_t* sv, uint32_t* out, cudaStream_t st,
                           bool sq = false) {
    const int nseg = (2 * Lv.n + Lv.b - 1) / Lv.b;
    const size_t smem = fused_smem_bytes(B, E, Lv.Lw, nseg, Lv.n, TOP);
    auto kern = k_fused_bottom<B, E, TOP>;
    // the C2 shape (level-1 parents of 65 limbs, b = 17) with compile-time offsets
    if constexpr (B == 4 && E == 18 && TOP == 0)
        if (Lv.n == 65 && Lv.b == 17 && Lv.Lw == 35 && g_its_static) kern = k_fused_bottom<4, 18, 0, 65, 17>;
    // the C3 / C4 bottom (parents of 66 limbs, b = 22)
    if constexpr (B == 3 && E == 23 && TOP == 0)
        if (Lv.n == 66 && Lv.b == 22 && Lv.Lw == 45 && g_its_static) kern = k_fused_bottom<3, 23, 0, 66, 22>;
    // squaring (v = u): the generic-shape kernel with the squaring base case
    // (instantiated for the base widths of C1-C5; others multiply u by u)
    bool sqk = false;
    if constexpr ((E == 18 || E == 23 || E == 33) && TOP != 3)
        if (sq) { kern = k_fused_bottom<B, E, TOP, 0, 0, true>; sqk = true; }
    static bool attr_set[3] = {false, false, false};   // per instantiation
    const int ai = sqk ? 2 : (kern == k_fused_bottom<B, E, TOP> ? 0 : 1);
    if (!attr_set[ai]) {
        if (const char* m = getenv("TOOM_DBG_FUSED_MASK")) {   // diagnostics only
            const int v = atoi(m);
            cudaMemcpyToSymbol(tg_fused_phase_mask, &v, sizeof v);
        }
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr_set[ai] = true;
    }
    const unsigned grid = (unsigned)((Lv.count + 31) / 32);
    kern<<<grid, 32 * (2 * B - 1), smem, st>>>(su, sv, out, Lv.count, Lv.n, Lv.b, Lv.Lw, 2 * Lv.n, nseg);
}

// mode: 0 interleaved signed parents, 1 row-major unsigned (top), 2 row-major signed
static toom_status launch_fused(const Level& Lv, int mode, const uint32_t* su, const uint32_t* sv, uint32_t* out,
                                cudaStream_t st, bool sq = false) {
    if (Lv.count == 0) return TOOM_OK;
    ProfScope ps(CAT_BASE, st);
#define TG_F(BB, EE)                                                      \
    if (Lv.B == BB && Lv.e == EE) {                                       \
        if (mode == 1) launch_fused_t<BB, EE, 1>(Lv, su, sv, out, st, sq);    \
        else if (mode == 2) launch_fused_t<BB, EE, 2>(Lv, su, sv, out, st, sq); \
        else if (mode == 3) launch_fused_t<BB, EE, 3>(Lv, su, sv, out, st, sq); \
        else launch_fused_t<BB, EE, 0>(Lv, su, sv, out, st, sq);              \
        ps.done(st);                                                      \
        ++t_launches;                                                     \
        return TOOM_OK;                                                   \
    }
    TG_F(3, 6) TG_F(3, 9) TG_F(3, 18) TG_F(3, 23) TG_F(3, 27) TG_F(3, 33)
    TG_F(4, 6) TG_F(4, 9) TG_F(4, 18) TG_F(4, 23) TG_F(4, 27) TG_F(4, 33)
#undef TG_F
    return TOOM_EUNSUPPORTED;
}

// a bottom level with the deferred denominator (csrc/fused_dc.cuh): B = 4 the
// C2 shape, B = 3 the bottom under the lazy levels
template <int B>
static toom_status launch_fused_dc(const Level& Lv, const uint32_t* su, const uint32_t* sv, uint32_t* out,
                                   cudaStream_t st) {
    if (Lv.count == 0) return TOOM_OK;
    ProfScope ps(CAT_BASE, st);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_fused_dc<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dc_smem_bytes<B>());
        cudaFuncSetAttribute(k_fused_dc<B>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    const unsigned grid = (unsigned)((Lv.count + 31) / 32);
    k_fused_dc<B><<<grid, 32 * (2 * B - 1), dc_smem_bytes<B>(), st>>>(su, sv, out, Lv.count);
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

// the C2 top level as one division over the common denominator (csrc/toplevel_cls.cuh)
static toom_status launch_interp_top_cls(const Level& Lv, const uint32_t* P1, uint32_t* w, bool def, cudaStream_t st) {
    if (Lv.count == 0) return TOOM_OK;
    ProfScope ps(CAT_INTERP, st);
    static bool attr[2] = {false, false};
    auto kern = def ? k_interp_top_cls<true> : k_interp_top_cls<false>;
    if (!attr[def]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cls_smem_bytes());
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr[def] = true;
    }
    const unsigned grid = (unsigned)((Lv.count + cls::G - 1) / cls::G);
    kern<<<grid, 32 * cls::NW, cls_smem_bytes(), st>>>(P1, w, Lv.count);
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

static bool g_disable_toprows = false;

static bool top_rows_ok(const Level& Lv) {
    if (g_disable_toprows || (Lv.B != 3 && Lv.B != 4)) return false;
    const int nseg = (2 * Lv.n + Lv.b - 1) / Lv.b;
    return interp_top_rows_smem(Lv.B, Lv.Lw, nseg) <= 200 * 1024 && Lv.Lw == 2 * Lv.b + 1;
}

static toom_status launch_eval_top_rows(const Level& Lv, const uint32_t* u, const uint32_t* v, uint32_t* U1,
                                        uint32_t* V1, cudaStream_t st, bool sq = false) {
    // 16-byte cp.async staging needs 16-byte aligned operand rows
    const bool v4 = g_eval_v4 && Lv.B <= 4 && (Lv.n & 3) == 0 && (Lv.b & 3) == 0 &&
                    ((((uintptr_t)u) | ((uintptr_t)v)) & 15) == 0;
    // squaring without the vectorised kernel: one thread per operand, u only
    if (sq && !v4) return launch_eval(Lv.B, true, u, nullptr, U1, nullptr, Lv.count, Lv.n, Lv.b, Lv.e, st);
    ProfScope ps(CAT_EVAL, st);
    const unsigned grid = (unsigned)((Lv.count + 31) / 32);
    if (v4 && sq && Lv.B == 3) k_eval_top_v4<3, true><<<grid, 32 * 5, 0, st>>>(u, u, U1, U1, Lv.count, Lv.n, Lv.b, Lv.e);
    else if (v4 && sq) k_eval_top_v4<4, true><<<grid, 32 * 7, 0, st>>>(u, u, U1, U1, Lv.count, Lv.n, Lv.b, Lv.e);
    else if (v4 && Lv.B == 3) k_eval_top_v4<3><<<grid, 32 * 5, 0, st>>>(u, v, U1, V1, Lv.count, Lv.n, Lv.b, Lv.e);
    else if (v4) k_eval_top_v4<4><<<grid, 32 * 7, 0, st>>>(u, v, U1, V1, Lv.count, Lv.n, Lv.b, Lv.e);
    else if (Lv.B == 3) k_eval_top_rows<3><<<grid, 32 * 5, 0, st>>>(u, v, U1, V1, Lv.count, Lv.n, Lv.b, Lv.e);
    else if (Lv.B == 4) k_eval_top_rows<4><<<grid, 32 * 7, 0, st>>>(u, v, U1, V1, Lv.count, Lv.n, Lv.b, Lv.e);
    else k_eval_top_rows<8><<<grid, 32 * 15, 0, st>>>(u, v, U1, V1, Lv.count, Lv.n, Lv.b, Lv.e);
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

template <int B>
static void launch_interp_top_rows_t(const Level& Lv, const uint32_t* P1, uint32_t* w, cudaStream_t st) {
    const int nseg = (2 * Lv.n + Lv.b - 1) / Lv.b;
    const size_t smem = interp_top_rows_smem(B, Lv.Lw, nseg);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_interp_top_rows<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(k_interp_top_rows<B>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr = true;
    }
    const unsigned grid = (unsigned)((Lv.count + 31) / 32);
    k_interp_top_rows<B><<<grid, 32 * (2 * B - 1), smem, st>>>(P1, w, Lv.count, 2 * Lv.e, Lv.Lw, Lv.b, 2 * Lv.n, nseg);
}


template <int B>
static bool launch_interp_top_smem_t(const Level& Lv, const uint32_t* P1, uint32_t* w, cudaStream_t st) {
    const int ywidth = 2 * Lv.e, nseg = (2 * Lv.n + Lv.b - 1) / Lv.b;
    constexpr int NP = 2 * B - 1;
    // instances per CTA: up to 32, two CTAs per SM if possible
    // instances per CTA: the shared-memory budget per CTA sets the occupancy
    // (2 CTAs per SM at ~113 KB)
    static const int budget_kb = [] {
        const char* e = getenv("TOOM_ITS_SMEM_KB");
        return e ? atoi(e) : 113;
    }();
    int G = 32;
    while (G > 4 && interp_top_smem_bytes(B, ywidth, G, nseg) > (size_t)budget_kb * 1024) G -= 4;
    if (interp_top_smem_bytes(B, ywidth, G, nseg) > 220 * 1024 || Lv.Lw >= ywidth || Lv.Lw != 2 * Lv.b + 1) return false;
    const size_t smem = interp_top_smem_bytes(B, ywidth, G, nseg);
    auto kern = k_interp_top_smem<B>;
    // the C2 shape (n = 256 limbs, b = 64) with compile-time offsets
    if constexpr (B == 4)
        if (ywidth == 130 && G == 28 && Lv.Lw == 129 && Lv.b == 64 && g_its_static) kern = k_interp_top_smem<4, 130, 28, 129, 64>;
    static bool attr[2] = {false, false};
    const int ai = kern == k_interp_top_smem<B> ? 0 : 1;
    if (!attr[ai]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
        cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        attr[ai] = true;
    }
    const unsigned grid = (unsigned)((Lv.count + G - 1) / G);
    kern<<<grid, 32 * NP, smem, st>>>(P1, w, Lv.count, ywidth, Lv.Lw, Lv.b, 2 * Lv.n, G, nseg);
    return true;
}

template <int B, int CH>
static void launch_interp_top_warp_t(const Level& Lv, const uint32_t* P1, uint32_t* w, cudaStream_t st) {
    const uint32_t o = B == 3 ? tg_combO_T3 : tg_combO_T4;
    WarpInterpConst K;
    K.o = o;
    K.oinv = B == 3 ? tg_combInv_T3 : tg_combInv_T4;
    K.sh = B == 3 ? tg_combS_T3 : tg_combS_T4;
    K.orcp = o > 1 ? ~0ull / o : 0ull;
    K.p32 = host_powmod(2, 32, o);
    K.Mch = host_powmod(2, 32ull * CH, o);
    K.mi = host_invmod(K.Mch, o);
    const int wpb = 8;
    const size_t smem = interp_top_warp_smem(B, 2 * Lv.e, CH, wpb);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_interp_top_warp<B, CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    const unsigned grid = (unsigned)((Lv.count + wpb - 1) / wpb);
    k_interp_top_warp<B, CH><<<grid, 32 * wpb, smem, st>>>(P1, w, Lv.count, 2 * Lv.e, Lv.b, 2 * Lv.n, K);
}

static void launch_interp_top_warp(const Level& Lv, const uint32_t* P1, uint32_t* w, cudaStream_t st) {
    const int ch = top_warp_ch(Lv);
#define TG_W(BB, CC) if (Lv.B == BB && ch == CC) launch_interp_top_warp_t<BB, CC>(Lv, P1, w, st);
    TG_W(3, 9) TG_W(3, 17) TG_W(3, 33) TG_W(4, 9) TG_W(4, 17) TG_W(4, 33)
#undef TG_W
}

static toom_status launch_interp_top_rows(const Level& Lv, const uint32_t* P1, uint32_t* w, cudaStream_t st) {
    ProfScope ps(CAT_INTERP, st);
    if (g_top_stream == 2) {
        const bool ok = Lv.B == 3 ? launch_interp_top_smem_t<3>(Lv, P1, w, st) : launch_interp_top_smem_t<4>(Lv, P1, w, st);
        if (ok) {
            ps.done(st);
            ++t_launches;
            return TOOM_OK;
        }
    }
    const int X = 2 * Lv.e - 2 * Lv.b;
    if (g_top_stream >= 1 && X >= 0 && X <= Lv.b) {
        const unsigned grid = (unsigned)((Lv.count + 32 * ITS_WARPS - 1) / (32 * ITS_WARPS));
        if (Lv.B == 3) k_interp_top_stream<3><<<grid, 32 * ITS_WARPS, 0, st>>>(P1, w, Lv.count, 2 * Lv.e, Lv.b, 2 * Lv.n);
        else k_interp_top_stream<4><<<grid, 32 * ITS_WARPS, 0, st>>>(P1, w, Lv.count, 2 * Lv.e, Lv.b, 2 * Lv.n);
        ps.done(st);
        ++t_launches;
        return TOOM_OK;
    }
    if (Lv.B == 3) launch_interp_top_rows_t<3>(Lv, P1, w, st);
    else launch_interp_top_rows_t<4>(Lv, P1, w, st);
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

// base level reached directly (no Toom level): schoolbook on row-major
// operands via a transposing copy
// row-major [count][n] -> interleaved [E][count], zero rows for n <= i < E
__global__ void k_transpose_in(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, size_t count, int n, int E,
                               int sgn) {
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= count * (size_t)E) return;
    const size_t c = gid / E;
    const int i = (int)(gid % E);
    uint32_t fill = 0;
    if (sgn && i >= n) fill = (src[c * (size_t)n + n - 1] >> 31) ? 0xFFFFFFFFu : 0u;
    dst[(size_t)i * count + c] = i < n ? src[c * (size_t)n + i] : fill;
}
__global__ void k_transpose_out(const uint32_t* __restrict__ src, uint32_t* __restrict__ dst, size_t count, int n2) {
    const size_t gid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (gid >= count * (size_t)n2) return;
    const size_t c = gid / n2;
    const int i = (int)(gid % n2);
    dst[gid] = src[(size_t)i * count + c];
}

// out[c][r] = in[r][c] for an R x C row-major matrix (32 x 32 smem tiles)
__global__ void k_transpose(const uint32_t* __restrict__ in, uint32_t* __restrict__ out, size_t R, size_t C) {
    __shared__ uint32_t tile[32][33];
    const size_t r0 = (size_t)blockIdx.y * 32, c0 = (size_t)blockIdx.x * 32;
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const size_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < R && c < C) tile[i][threadIdx.x] = in[r * C + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += blockDim.y) {
        const size_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < R && c < C) out[c * R + r] = tile[threadIdx.x][i];
    }
}

static void launch_transpose(const uint32_t* in, uint32_t* out, size_t R, size_t C, cudaStream_t st) {
    dim3 grid((unsigned)((C + 31) / 32), (unsigned)((R + 31) / 32));
    k_transpose<<<grid, dim3(32, 8), 0, st>>>(in, out, R, C);
    ++t_launches;
}

// ------------------------------------------------------------------------
// long-vector levels: op descriptors for one call (down: evaluation of both
// operands at every point; up: the interpolation program, then the
// recomposition op), built on the host and uploaded once per call
// ------------------------------------------------------------------------
struct LongCall {
    std::vector<LOpDev> down, up;        // single-output ops (per level, in launch order)
    std::vector<LMultiDev> mdown, mup;   // multi-output ops
    std::vector<LBigDev> bup;            // wide-multiplier multi-output ops (matrix-form T16)
    // launch order of a level: (kind 0 = op, 1 = multi, 3 = big, index into the level's vectors)
    std::vector<std::pair<int, int>> sdown, sup;
};


// layout of level l's child operand / product families
static LVec child_vec(const Plan& plan, size_t l, const uint8_t* ws, size_t off, int width, int k) {
    const Level& L = plan.lv[l];
    if ((int)l == plan.bnd) {   // row-major staging, transposed to/from the level below
        size_t o = plan.offT;
        if (off == L.offV && L.offV != L.offU) o += (size_t)L.e * L.count * L.npts * 4;
        const uint32_t* base = (const uint32_t*)(ws + o);
        return LVec{base + (size_t)k * L.count * width, width, 1, width, 1};
    }
    const bool next_fused = plan.fused && l + 1 == plan.lv.size() - 2;
    const bool next_long = (l + 1 < plan.lv.size() - 1) && (plan.lv[l + 1].lng || next_fused);
    const uint32_t* base = (const uint32_t*)(ws + off);
    if (next_long)   // row-major [npts*count][width], child k*count + c
        return LVec{base + (size_t)k * L.count * width, width, 1, width, 1};
    // interleaved [width][npts*count]
    return LVec{base + (size_t)k * L.count, 1, (long long)L.npts * (long long)L.count, width, 1};
}

// evaluation ops of one long level: U(x_k) for every point k of one operand
// family `par` (Eq. 1.1 split as slices, homogeneous point values)
template <class ChildF>
static void long_eval_ops(const Level& L, const LVec& par, ChildF child, std::vector<LOpDev>& out, int k0 = 0,
                          int k1 = INT_MAX) {
    LongTables T;
    long_tables(L.B, T);
    for (int k = 0; k < T.neo; ++k) {
        const tg_lop& o = T.eo[k];
        if (o.dst < k0 || o.dst >= k1) continue;   // (a range of points: the sharded top level)
        LVec dv = child(o.dst - k0);
        LOpBuilder b((uint32_t*)dv.base, dv.is, dv.ls, L.e, (int)L.count);
        for (int t = 0; t < o.nt; ++t) {
            const tg_lterm& tm = T.et[o.t0 + t];
            const int j = -tm.src - 1;
            const int len = (j == L.B - 1) ? L.lentop : L.b;
            b.add(par, tm.m, tm.s, j * L.b, len, (j == L.B - 1) ? -1 : 0);
        }
        b.op.wide = o.wide;
        out.push_back(b.op);
    }
}

// interpolation program (steps a4) over the slot pool, then the
// recomposition w = sum_j w_j 2^(32 b j) (Eq. 1.3, step a5) into dst
// (row-major [count][2n], two's complement)
static bool g_long_comb = true;   // T3/T4 long levels: one combined interp+recompose op

template <class YF>
static void long_interp_ops(const Level& L, YF yv, uint32_t* slots, uint32_t* dst, std::vector<LOpDev>& out) {
    LongTables T;
    long_tables(L.B, T);
    const int cnt = (int)L.count;
    if (g_long_comb && (L.B == 3 || L.B == 4) && L.Lw == 2 * L.b + 1) {
        // Dc w = sum_j 2^(32 b j) sum_k A'_jk y_k, then / Dc (Eq. 1.3)
        const long long* A = L.B == 3 ? &tg_lcomb_T3[0][0] : &tg_lcomb_T4[0][0];
        const uint32_t o = L.B == 3 ? tg_lcombO_T3 : tg_lcombO_T4;
        const int sh = L.B == 3 ? tg_lcombS_T3 : tg_lcombS_T4;
        LOpBuilder b(dst, 2 * L.n, 1, 2 * L.n, cnt, o, sh);
        for (int j = 0; j < L.npts; ++j)
            for (int k = 0; k < L.npts; ++k)
                if (A[j * L.npts + k]) b.add(yv(k), A[j * L.npts + k], 32ll * L.b * j);
        b.op.wide = 0;
        out.push_back(b.op);
        return;
    }
    const int Wt = long_Wt(L);
    auto slot_vec = [&](int sl) { return LVec{slots + (size_t)sl * cnt * Wt, Wt, 1, Wt, 0}; };
    for (int i = 0; i < T.nio; ++i) {
        const tg_lop& o = T.io[i];
        LVec dv = slot_vec(o.dst);
        LOpBuilder b((uint32_t*)dv.base, dv.is, dv.ls, Wt, cnt, o.odiv, o.shr);
        for (int t = 0; t < o.nt; ++t) {
            const tg_lterm& tm = T.it[o.t0 + t];
            b.add(tm.src < 0 ? yv(-tm.src - 1) : slot_vec(tm.src), tm.m, tm.s);
        }
        b.op.wide = o.wide;
        out.push_back(b.op);
    }
    LOpBuilder b(dst, 2 * L.n, 1, 2 * L.n, cnt);
    for (int j = 0; j < L.npts; ++j) {
        const int src = T.iout[j];
        if (src < 0) b.add(yv(-src - 1), 1, 32ll * L.b * j);
        else b.add(slot_vec(src), 1, 32ll * L.b * j, 0, L.Lw, 1);
    }
    b.op.wide = 0;
    out.push_back(b.op);
}

// tile shape of a multi-output op: the largest tile within the shared-memory
// budget that pads the vector by at most 1/8
// multi-output ops staging at least this many sources use 4 limbs per thread
// (16: the Toom-16 evaluation, whose 16 staged sources leave a 16-limb tile 2
// warps per CTA; C5 69.36 ms at 16 limbs, 68.74 ms with 4 from 16 sources,
// 69.23 ms with 4 from 8 sources, gpurun_out/ch4_time.log of round 2)
static int g_multi_ch4_ns = [] {
    const char* e = getenv("TOOM_MULTI_CH4_NS");
    return e ? atoi(e) : 16;
}();

static bool multi_shape(LMultiDev& d) {
    d.ch = d.ns >= g_multi_ch4_ns ? 4 : 16;   // 16: the per-output scan amortised over 16 limbs
    int best = 0;
    long long bestw = -1;
    for (int nt = LV_NT; nt >= 32; nt -= 32) {
        if (long_multi_smem(nt, d.ch, d.ns) > 96 * 1024) continue;
        const long long tl = (long long)nt * d.ch, tiles = (d.W + tl - 1) / tl, pad = tiles * tl;
        if (pad * 8 <= (long long)d.W * 9) { best = nt; break; }
        if (bestw < 0 || pad < bestw) { bestw = pad; best = nt; }
    }
    if (!best) return false;
    d.nthreads = best;
    d.tiles_per_inst = (d.W + best * d.ch - 1) / (best * d.ch);
    return true;
}

static void multi_out(LMOut& O, uint32_t* dst, uint32_t o, int shr, int ch) {
    memset(&O, 0, sizeof O);
    O.dst = dst;
    O.o = o;
    O.oinv = host_inv32(o);
    if (o > 1) {
        O.orcp = ~0ull / o;
        O.p32 = host_powmod(2, 32, o);
        O.Mch = host_powmod(2, 32ull * ch, o);
        O.mi = host_invmod(O.Mch, o);
    }
    O.sa = shr / 32;
    O.sr = shr % 32;
}

static bool g_long_meval = true;

// evaluation of a long level: all 2B-1 points of one operand family (sources:
// the B blocks of Eq. 1.1; multipliers p^j q^(n-j))
template <class ChildF>
static bool long_multi_eval(const Level& L, const LVec& par, ChildF child, LMultiDev& d) {
    LongTables T;
    long_tables(L.B, T);
    if (!g_long_meval || L.B > LM_MAXS || L.npts > LM_MAXO || par.ls != 1) return false;
    memset(&d, 0, sizeof d);
    d.ns = L.B;
    d.no = L.npts;
    d.W = L.e;
    d.count = (int)L.count;
    for (int j = 0; j < L.B; ++j) {
        const int len = (j == L.B - 1) ? L.lentop : L.b;
        d.src[j] = LMSrc{par.base + (size_t)j * L.b, par.is, len, (j == L.B - 1) ? par.sign : 0};
    }
    for (int k = 0; k < T.neo; ++k) {
        const tg_lop& o = T.eo[k];
        for (int t = 0; t < o.nt; ++t) {
            const tg_lterm& tm = T.et[o.t0 + t];
            d.m[o.dst][-tm.src - 1] += tm.m * (1ll << tm.s);
        }
    }
    unsigned long long sum = 0;
    for (int k = 0; k < L.npts; ++k) {
        unsigned long long r = 0;
        for (int j = 0; j < L.B; ++j) r += (unsigned long long)(d.m[k][j] < 0 ? -d.m[k][j] : d.m[k][j]);
        sum = std::max(sum, r);
    }
    d.wide = sum >= (1ull << 30);
    if (!multi_shape(d)) return false;
    for (int k = 0; k < L.npts; ++k) {
        const LVec c = child(k);
        if (c.ls != 1 && k == 0) { /* interleaved children are fine: strided stores */ }
        multi_out(d.out[k], (uint32_t*)c.base, 1, 0, d.ch);
        d.dst_is = c.is;
        d.dst_ls = c.ls;
    }
    return true;
}

// interpolation rows of a Toom-3/4 long level: w_j = (sum_k A_jk y_k)/D_j for
// the interior rows j = 1 .. 2B-3 (w_0 = y_0, w_2n = y_inf), into the slots
template <class YF>
static bool long_multi_rows(const Level& L, YF yv, uint32_t* slots, LMultiDev& d) {
    if (!g_long_meval || (L.B != 3 && L.B != 4) || L.Lw != 2 * L.b + 1) return false;
    const long long* A = L.B == 3 ? &tg_lrowA_T3[0][0] : &tg_lrowA_T4[0][0];
    const unsigned* O = L.B == 3 ? tg_lrowO_T3 : tg_lrowO_T4;
    const int* S = L.B == 3 ? tg_lrowS_T3 : tg_lrowS_T4;
    memset(&d, 0, sizeof d);
    d.ns = L.npts;
    d.no = L.npts - 2;
    d.W = L.Lw;
    d.count = (int)L.count;
    for (int k = 0; k < L.npts; ++k) {
        const LVec y = yv(k);
        if (y.ls != 1) return false;
        d.src[k] = LMSrc{y.base, y.is, 2 * L.e, 1};
    }
    for (int j = 1; j <= L.npts - 2; ++j)
        for (int k = 0; k < L.npts; ++k) d.m[j - 1][k] = A[j * L.npts + k];
    d.wide = 0;
    if (!multi_shape(d)) return false;
    for (int j = 1; j <= L.npts - 2; ++j)
        multi_out(d.out[j - 1], slots + (size_t)(j - 1) * L.count * L.Lw, O[j], S[j], d.ch);
    d.dst_is = L.Lw;
    d.dst_ls = 1;
    return true;
}

// ---- matrix-form Toom-16 interpolation: the
// even-odd split (Eqs. 4.5-4.6), one dense pass per half with wide
// multipliers (the symbolic inverse, gen/toomgen.py t16_matrix_form), the
// exact divisions by the remaining coprime word factors of each row's
// denominator, and the recomposition (Eq. 1.3).
static void big_out(LBigDev& d) {
    d.ch = LB_CH;
    d.nthreads = 128;
    d.tiles_per_inst = (d.W + d.nthreads * LB_CH - 1) / (d.nthreads * LB_CH);
}

template <class YF>
static void long_t16_matrix(const Level& L, YF yv, uint32_t* slots, uint32_t* dst, LongCall& lc) {
    const int cnt = (int)L.count, Wt = long_Wt(L), W2 = 2 * L.e, Lw = L.Lw;
    auto slot = [&](int g, int i) { return slots + (size_t)(g * 15 + i) * cnt * Wt; };   // groups E=0 O=1 R=2 T=3, y' = 60
    uint32_t* Y = slots + (size_t)60 * cnt * Wt;
    constexpr int NPR = tg_f1_npairs;
    auto msrc = [&](const uint32_t* base, int len) { return LMSrc{base, (long long)Wt, len, 1}; };
    auto ysrc = [&](int k) {
        const LVec y = yv(k);
        return LMSrc{y.base, y.is, 2 * L.e, 1};
    };
    // 1. E_i = y+ + y-, O_i = y+ - y- (two multi ops of 7 pairs)
    for (int h = 0; h < 2; ++h) {
        LMultiDev d;
        memset(&d, 0, sizeof d);
        const int p0 = h * 7, np = std::min(7, NPR - p0);
        d.ns = 2 * np;
        d.no = 2 * np;
        d.W = W2 + 1;
        d.count = cnt;
        for (int i = 0; i < np; ++i) {
            d.src[2 * i] = ysrc(tg_f1_pair[p0 + i][0]);
            d.src[2 * i + 1] = ysrc(tg_f1_pair[p0 + i][1]);
            d.m[2 * i][2 * i] = 1;
            d.m[2 * i][2 * i + 1] = 1;
            d.m[2 * i + 1][2 * i] = 1;
            d.m[2 * i + 1][2 * i + 1] = -1;
        }
        multi_shape(d);
        for (int i = 0; i < np; ++i) {
            multi_out(d.out[2 * i], slot(0, p0 + i), 1, 0, d.ch);
            multi_out(d.out[2 * i + 1], slot(1, p0 + i), 1, 0, d.ch);
        }
        d.dst_is = Wt;
        d.dst_ls = 1;
        lc.sup.push_back({1, (int)lc.mup.size()});
        lc.mup.push_back(d);
    }
    // exact division of rows `nr` in group gs by their word factor f, into group gd
    auto div_pass = [&](int nr, int gs, int gd, const unsigned (*o)[3], int f) {
        LMultiDev d;
        memset(&d, 0, sizeof d);
        d.ns = d.no = nr;
        d.W = Lw;
        d.count = cnt;
        for (int r = 0; r < nr; ++r) {
            d.src[r] = msrc(slot(gs, r), Lw);
            d.m[r][r] = 1;
        }
        multi_shape(d);
        for (int r = 0; r < nr; ++r) multi_out(d.out[r], slot(gd, r), o[r][f], 0, d.ch);
        d.dst_is = Wt;
        d.dst_ls = 1;
        lc.sup.push_back({1, (int)lc.mup.size()});
        lc.mup.push_back(d);
    };
    auto big_rows = [&](int nr, int ns, const LMSrc* src, const int (*a)[17][4], int astride, const unsigned (*o)[3],
                        const int* sh, int gd) {
        (void)astride;
        LBigDev d;
        memset(&d, 0, sizeof d);
        d.ns = ns;
        d.no = nr;
        d.W = Lw;
        d.count = cnt;
        for (int sI = 0; sI < ns; ++sI) d.src[sI] = src[sI];
        for (int r = 0; r < nr; ++r)
            for (int sI = 0; sI < ns; ++sI) {
                int nd = 0;
                for (int k = 0; k < LB_ND; ++k) {
                    d.a[r][sI][k] = a[r][sI][k];
                    if (a[r][sI][k]) nd = k + 1;
                }
                d.nd[r][sI] = nd;
            }
        big_out(d);
        for (int r = 0; r < nr; ++r) multi_out(d.out[r], slot(gd, r), o[r][0], sh[r], LB_CH);
        d.dst_is = Wt;
        d.dst_ls = 1;
        lc.sup.push_back({3, (int)lc.bup.size()});
        lc.bup.push_back(d);
    };
    // 2. even rows (sources E_0..13, y_0, y_inf), then the remaining word factors
    {
        static int ae[tg_f1_even_n][17][4];
        for (int r = 0; r < tg_f1_even_n; ++r)
            for (int sI = 0; sI < 17; ++sI)
                for (int k = 0; k < 4; ++k) ae[r][sI][k] = sI < NPR + 2 ? tg_f1_even_a[r][sI][k] : 0;
        LMSrc src[LB_MAXS];
        for (int i = 0; i < NPR; ++i) src[i] = msrc(slot(0, i), W2 + 1);
        src[NPR] = ysrc(tg_f1_i0);
        src[NPR + 1] = ysrc(tg_f1_iinf);
        big_rows(tg_f1_even_n, NPR + 2, src, ae, 17, tg_f1_even_o, tg_f1_even_s, 2);
        div_pass(tg_f1_even_n, 2, 3, tg_f1_even_o, 1);
        div_pass(tg_f1_even_n, 3, 2, tg_f1_even_o, 2);   // even w_2..w_28 in group R
    }
    // 3. y' = y(2:5) - sum_{j even} w_j 2^j 5^(30-j)
    {
        LBigDev d;
        memset(&d, 0, sizeof d);
        d.ns = 2 + tg_f1_even_n + 1;
        d.no = 1;
        d.W = W2 + 1;
        d.count = cnt;
        d.src[0] = ysrc(tg_f1_iu);
        d.a[0][0][0] = 1;
        d.nd[0][0] = 1;
        for (int jj = 0; jj <= tg_f1_even_n + 1; ++jj) {   // w_0, w_2 .. w_28, w_30
            LMSrc sI = jj == 0 ? ysrc(tg_f1_i0) : (jj == tg_f1_even_n + 1 ? ysrc(tg_f1_iinf) : msrc(slot(2, jj - 1), Lw));
            d.src[1 + jj] = sI;
            int nd = 0;
            for (int k = 0; k < LB_ND; ++k) {
                d.a[0][1 + jj][k] = -tg_f1_ymul[jj][k];
                if (tg_f1_ymul[jj][k]) nd = k + 1;
            }
            d.nd[0][1 + jj] = nd;
        }
        big_out(d);
        multi_out(d.out[0], Y, 1, 0, LB_CH);
        d.dst_is = Wt;
        d.dst_ls = 1;
        lc.sup.push_back({3, (int)lc.bup.size()});
        lc.bup.push_back(d);
    }
    // 4. odd rows (sources O_0..13, y'), then the remaining word factors
    {
        static int ao[tg_f1_odd_n][17][4];
        for (int r = 0; r < tg_f1_odd_n; ++r)
            for (int sI = 0; sI < 17; ++sI)
                for (int k = 0; k < 4; ++k) ao[r][sI][k] = sI < NPR + 1 ? tg_f1_odd_a[r][sI][k] : 0;
        LMSrc src[LB_MAXS];
        for (int i = 0; i < NPR; ++i) src[i] = msrc(slot(1, i), W2 + 1);
        src[NPR] = msrc(Y, W2 + 1);
        big_rows(tg_f1_odd_n, NPR + 1, src, ao, 17, tg_f1_odd_o, tg_f1_odd_s, 3);
        div_pass(tg_f1_odd_n, 3, 0, tg_f1_odd_o, 1);
        div_pass(tg_f1_odd_n, 0, 3, tg_f1_odd_o, 2);     // odd w_1..w_29 in group T
    }
    // 5. w = sum_j w_j 2^(32 b j)
    LOpBuilder b(dst, 2 * L.n, 1, 2 * L.n, cnt);
    for (int j = 0; j <= 30; ++j) {
        if (j == 0) b.add(yv(tg_f1_i0), 1, 0);
        else if (j == 30) b.add(yv(tg_f1_iinf), 1, 32ll * L.b * j);
        else {
            const int g = (j & 1) ? 3 : 2, r = (j & 1) ? (j - 1) / 2 : (j - 2) / 2;
            b.add(LVec{slot(g, r), Wt, 1, Wt, 0}, 1, 32ll * L.b * j, 0, Lw, 1);
        }
    }
    b.op.wide = 0;
    lc.sup.push_back({0, (int)lc.up.size()});
    lc.up.push_back(b.op);
}

static void build_long_level(const Plan& plan, size_t l, uint32_t* w, const uint32_t* u, const uint32_t* v, uint8_t* ws,
                             LongCall& lc) {
    const Level& L = plan.lv[l];
    for (int opd = 0; opd < (plan.square ? 1 : 2); ++opd) {   // squaring: V = U
        LVec par;
        if (l == 0) par = LVec{opd ? v : u, L.n, 1, L.n, plan.signed_in ? 1 : 0};   // user operands, row-major
        else par = LVec{(const uint32_t*)(ws + (opd ? plan.lv[l - 1].offV : plan.lv[l - 1].offU)), L.n, 1, L.n, 1};
        const size_t off = opd ? L.offV : L.offU;
        auto child = [&](int k) { return child_vec(plan, l, ws, off, L.e, k); };
        LMultiDev d;
        if (long_multi_eval(L, par, child, d)) {
            lc.sdown.push_back({1, (int)lc.mdown.size()});
            lc.mdown.push_back(d);
        } else {
            const size_t a = lc.down.size();
            long_eval_ops(L, par, child, lc.down);
            for (size_t i = a; i < lc.down.size(); ++i) lc.sdown.push_back({0, (int)i});
        }
    }
    uint32_t* dst = (l == 0) ? w : (uint32_t*)(ws + plan.lv[l - 1].offP);
    uint32_t* slots = (uint32_t*)(ws + plan.offSlots);
    auto yv = [&](int k) { return child_vec(plan, l, ws, L.offP, 2 * L.e, k); };
    LMultiDev d;
    if (long_multi_rows(L, yv, slots, d)) {
        // rows w_1 .. w_2n-1 into the slots, then w = sum_j w_j 2^(32 b j)
        lc.sup.push_back({1, (int)lc.mup.size()});
        lc.mup.push_back(d);
        LOpBuilder b(dst, 2 * L.n, 1, 2 * L.n, (int)L.count);
        for (int j = 0; j < L.npts; ++j) {
            if (j == 0 || j == L.npts - 1) b.add(yv(j), 1, 32ll * L.b * j);
            else b.add(LVec{slots + (size_t)(j - 1) * L.count * L.Lw, L.Lw, 1, L.Lw, 1}, 1, 32ll * L.b * j);
        }
        b.op.wide = 0;
        lc.sup.push_back({0, (int)lc.up.size()});
        lc.up.push_back(b.op);
        return;
    }
    // (the matrix form stages its sources row-major: products of a schoolbook
    // level directly below, interleaved, take the Newton program)
    if (L.B == 16 && g_t16_matrix && yv(0).ls == 1) {
        long_t16_matrix(L, yv, slots, dst, lc);
        return;
    }
    const size_t a = lc.up.size();
    long_interp_ops(L, yv, slots, dst, lc.up);
    for (size_t i = a; i < lc.up.size(); ++i) lc.sup.push_back({0, (int)i});
}

static std::mutex g_desc_mu;
static LOpDev* g_desc_host = nullptr;   // pinned staging for the descriptor upload
static size_t g_desc_cap = 0;
static cudaEvent_t g_desc_ev = nullptr;

// upload the call's op descriptors (pinned staging, one copy per kind) and
// reset the scan status / tile counters, all stream-ordered
static toom_status long_prepare(const std::vector<LOpDev>& ops, const std::vector<LMultiDev>& mops, LOpDev* ddesc,
                                LMultiDev* mdesc, LStatus* status, size_t nStatus, unsigned* ctr, size_t nCtr,
                                cudaStream_t st, const std::vector<LBigDev>* bops = nullptr, LBigDev* bdesc = nullptr) {
    const size_t nd = ops.size(), ne = mops.size(), nb = bops ? bops->size() : 0;
    const size_t bytes = nd * sizeof(LOpDev) + ne * sizeof(LMultiDev) + nb * sizeof(LBigDev);
    std::lock_guard<std::mutex> g(g_desc_mu);
    if (g_desc_ev) cudaEventSynchronize(g_desc_ev);   // previous upload finished reading the staging
    if (bytes > g_desc_cap * sizeof(LOpDev)) {
        if (g_desc_host) cudaFreeHost(g_desc_host);
        const size_t cap = (bytes + sizeof(LOpDev) - 1) / sizeof(LOpDev);
        if (cudaMallocHost((void**)&g_desc_host, cap * sizeof(LOpDev)) != cudaSuccess) {
            cudaGetLastError();
            g_desc_host = nullptr;
            g_desc_cap = 0;
            return TOOM_ENOMEM;
        }
        g_desc_cap = cap;
    }
    if (nd) {
        memcpy(g_desc_host, ops.data(), nd * sizeof(LOpDev));
        if (cudaMemcpyAsync(ddesc, g_desc_host, nd * sizeof(LOpDev), cudaMemcpyHostToDevice, st) != cudaSuccess)
            return TOOM_ECUDA;
    }
    if (ne) {
        uint8_t* hb = (uint8_t*)(g_desc_host + nd);
        memcpy(hb, mops.data(), ne * sizeof(LMultiDev));
        if (cudaMemcpyAsync(mdesc, hb, ne * sizeof(LMultiDev), cudaMemcpyHostToDevice, st) != cudaSuccess)
            return TOOM_ECUDA;
    }
    if (nb) {
        uint8_t* hb = (uint8_t*)(g_desc_host + nd) + ne * sizeof(LMultiDev);
        memcpy(hb, bops->data(), nb * sizeof(LBigDev));
        if (cudaMemcpyAsync(bdesc, hb, nb * sizeof(LBigDev), cudaMemcpyHostToDevice, st) != cudaSuccess)
            return TOOM_ECUDA;
    }
    if (!g_desc_ev) cudaEventCreateWithFlags(&g_desc_ev, cudaEventDisableTiming);
    cudaEventRecord(g_desc_ev, st);
    cudaMemsetAsync(status, 0, nStatus * sizeof(LStatus), st);
    cudaMemsetAsync(ctr, 0, nCtr * sizeof(unsigned), st);
    return TOOM_OK;
}

// single-pass decoupled look-back executor (longvec.cuh) instead of the
// two-pass one (longvec2.cuh): TOOM_LONG_LOOKBACK=1, for comparison only
static const bool g_long_lookback = [] {
    const char* e = getenv("TOOM_LONG_LOOKBACK");
    return e ? atoi(e) != 0 : false;
}();

// one two-pass op: summaries, scan, finish (longvec2.cuh)
static void launch_scan2(LTile* tiles, int count, int tpi, int no, int nthreads, const uint32_t* o,
                         const unsigned long long* orcp, const uint32_t* mch, const uint32_t* mi, cudaStream_t st) {
    L2ScanArgs A;
    memset(&A, 0, sizeof A);
    A.tiles = tiles;
    A.count = count;
    A.tpi = tpi;
    A.no = no;
    A.nthreads = nthreads;
    for (int i = 0; i < no; ++i) { A.o[i] = o[i]; A.orcp[i] = orcp[i]; A.mch[i] = mch[i]; A.mi[i] = mi[i]; }
    const size_t warps = (size_t)count * no;
    if (tpi >= 128) k_lscan2_blk<<<(unsigned)warps, 1024, 0, st>>>(A);   // one CTA per vector
    else k_lscan2<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(A);
    ++t_launches;
}

static toom_status launch_long_multi(const LMultiDev& d, const LMultiDev* dd, LStatus* status, unsigned* ctr,
                                     unsigned& epoch, int cat, cudaStream_t st) {
    const unsigned grid = (unsigned)((size_t)d.count * d.tiles_per_inst);
    if (grid == 0) return TOOM_OK;
    ProfScope ps(cat, st);
    if (!g_long_lookback) {
        const size_t sm = lmulti2_smem(d.nthreads, d.ch, d.ns);
        LTile* tiles = reinterpret_cast<LTile*>(status);
        const bool one = d.tiles_per_inst == 1;   // the tile is the whole vector: one pass
#define TG_LM2(W, C)                                                                                      \
        {                                                                                                 \
            static bool attr = false;                                                                     \
            if (!attr) {                                                                                  \
                cudaFuncSetAttribute(k_lmulti2<W, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
                attr = true;                                                                              \
            }                                                                                             \
            if (one) {                                                                                    \
                k_lmulti2<W, C><<<grid, d.nthreads, sm, st>>>(dd, tiles, 3);                              \
            } else {                                                                                      \
                k_lmulti2<W, C><<<grid, d.nthreads, sm, st>>>(dd, tiles, 1);                              \
                launch_scan2(tiles, d.count, d.tiles_per_inst, d.no, d.nthreads, o, orcp, mch, mi, st);   \
                k_lmulti2<W, C><<<grid, d.nthreads, sm, st>>>(dd, tiles, 2);                              \
            }                                                                                             \
        }
        uint32_t o[LM_MAXO], mch[LM_MAXO], mi[LM_MAXO];
        unsigned long long orcp[LM_MAXO];
        for (int i = 0; i < d.no; ++i) { o[i] = d.out[i].o; orcp[i] = d.out[i].orcp; mch[i] = d.out[i].Mch; mi[i] = d.out[i].mi; }
        if (d.ch == 16) {
            if (d.wide) TG_LM2(true, 16) else TG_LM2(false, 16)
        } else {
            if (d.wide) TG_LM2(true, 4) else TG_LM2(false, 4)
        }
#undef TG_LM2
        ps.done(st);
        t_launches += one ? 0 : 2;
        return TOOM_OK;
    }
    const size_t sm = long_multi_smem(d.nthreads, d.ch, d.ns);
#define TG_LM(W, C)                                                                                        \
    {                                                                                                      \
        static bool attr = false;                                                                          \
        if (!attr) {                                                                                       \
            cudaFuncSetAttribute(k_long_multi<W, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
            attr = true;                                                                                   \
        }                                                                                                  \
        k_long_multi<W, C><<<grid, d.nthreads, sm, st>>>(dd, status, epoch, ctr);                         \
    }
    if (d.ch == 16) {
        if (d.wide) TG_LM(true, 16) else TG_LM(false, 16)
    } else {
        if (d.wide) TG_LM(true, 4) else TG_LM(false, 4)
    }
#undef TG_LM
    ps.done(st);
    ++epoch;
    ++t_launches;
    return TOOM_OK;
}

// wide-multiplier multi-output op (matrix-form T16): two passes + scan, or
// one pass when a tile holds the whole vector
static toom_status launch_long_big(const LBigDev& d, const LBigDev* dd, LStatus* status, int cat, cudaStream_t st) {
    const unsigned grid = (unsigned)((size_t)d.count * d.tiles_per_inst);
    if (grid == 0) return TOOM_OK;
    ProfScope ps(cat, st);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_lbig2, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        attr = true;
    }
    const size_t sm = lbig2_smem(d.nthreads, d.ns);
    LTile* tiles = reinterpret_cast<LTile*>(status);
    if (d.tiles_per_inst == 1) {
        k_lbig2<<<grid, d.nthreads, sm, st>>>(dd, tiles, 3);
    } else {
        uint32_t o[LM_MAXO], mch[LM_MAXO], mi[LM_MAXO];
        unsigned long long orcp[LM_MAXO];
        for (int i = 0; i < d.no; ++i) { o[i] = d.out[i].o; orcp[i] = d.out[i].orcp; mch[i] = d.out[i].Mch; mi[i] = d.out[i].mi; }
        k_lbig2<<<grid, d.nthreads, sm, st>>>(dd, tiles, 1);
        launch_scan2(tiles, d.count, d.tiles_per_inst, d.no, d.nthreads, o, orcp, mch, mi, st);
        k_lbig2<<<grid, d.nthreads, sm, st>>>(dd, tiles, 2);
        t_launches += 2;
    }
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

// long ops with at least this many tiles per instance use the two-pass scan
static int g_two_pass_tiles = [] {
    const char* e = getenv("TOOM_TWO_PASS_TILES");
    return e ? atoi(e) : 1 << 30;   // off by default: measured slower (C4 7.4 -> 18 ms at 64)
}();

static toom_status launch_long_ops(const std::vector<LOpDev>& ops, size_t first, const LOpDev* ddesc, LStatus* status,
                                   unsigned* ctr, unsigned& epoch, int cat, cudaStream_t st) {
    for (size_t i = 0; i < ops.size(); ++i) {
        const LOpDev& o = ops[i];
        const unsigned grid = (unsigned)((size_t)o.count * o.tiles_per_inst);
        if (grid == 0) continue;
        ProfScope ps(cat, st);
        const LOpDev* d = ddesc + first + i;
        unsigned* cp = ctr + first + i;
        const size_t qs = ((size_t)o.nthreads * o.ch + LV_MAXHALO + 1 + (size_t)(o.ch + 1) * (o.nthreads + 1)) * 4;
        if (!g_long_lookback) {
            LTile* tiles = reinterpret_cast<LTile*>(status);
            static bool attr2 = false;
            if (!attr2) {
                cudaFuncSetAttribute(k_lop2<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
                cudaFuncSetAttribute(k_lop2<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
                cudaFuncSetAttribute(k_lop2<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
                cudaFuncSetAttribute(k_lop2<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
                attr2 = true;
            }
            const size_t qs2 = lop2_smem(o.nthreads, o.ch);
            const bool one = o.tiles_per_inst == 1;   // the tile is the whole vector: one pass
            for (int ph = one ? 3 : 1; ph <= (one ? 3 : 2); ++ph) {
                if (ph == 2) {
                    const unsigned long long orcp = o.orcp;
                    launch_scan2(tiles, o.count, o.tiles_per_inst, 1, o.nthreads, &o.o, &orcp, &o.Mch, &o.mi, st);
                }
                if (o.ch == 16) {
                    if (o.wide) k_lop2<true, 16><<<grid, o.nthreads, qs2, st>>>(d, tiles, ph);
                    else k_lop2<false, 16><<<grid, o.nthreads, qs2, st>>>(d, tiles, ph);
                } else {
                    if (o.wide) k_lop2<true, 4><<<grid, o.nthreads, qs2, st>>>(d, tiles, ph);
                    else k_lop2<false, 4><<<grid, o.nthreads, qs2, st>>>(d, tiles, ph);
                }
            }
            ps.done(st);
            t_launches += one ? 0 : 2;
            continue;
        }
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute(k_long_op<true, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
            cudaFuncSetAttribute(k_long_op<false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
            cudaFuncSetAttribute(k_long_op<true, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
            cudaFuncSetAttribute(k_long_op<false, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
            attr = true;
        }
        // many tiles per vector: two-pass scan (aggregates, one scan CTA per
        // instance, finish) instead of the latency-bound look-back chain
        const bool two = o.tiles_per_inst >= g_two_pass_tiles;
        for (int ph = two ? 1 : 0; ph <= (two ? 2 : 0); ++ph) {
            if (ph == 2) {
                k_long_scan<<<o.count, 1024, 0, st>>>(status, o.tiles_per_inst, o.o, o.orcp);
                ++t_launches;
            }
            if (o.ch == 16) {
                if (o.wide) k_long_op<true, 16><<<grid, o.nthreads, qs, st>>>(d, status, epoch, cp, ph);
                else k_long_op<false, 16><<<grid, o.nthreads, qs, st>>>(d, status, epoch, cp, ph);
            } else {
                if (o.wide) k_long_op<true, 4><<<grid, o.nthreads, qs, st>>>(d, status, epoch, cp, ph);
                else k_long_op<false, 4><<<grid, o.nthreads, qs, st>>>(d, status, epoch, cp, ph);
            }
            if (ph == 1) ++t_launches;
        }
        ps.done(st);
        ++epoch;
        ++t_launches;
    }
    return TOOM_OK;
}

// one instance-resident level (level34.cuh): evaluation (down) or
// interpolation + recomposition (up), one CTA per instance, row-major layouts
static toom_status launch_res(const Plan& plan, size_t l, bool down, uint32_t* w, const uint32_t* u, const uint32_t* v,
                              uint8_t* ws, cudaStream_t st) {
    const Level& L = plan.lv[l];
    if (L.count == 0) return TOOM_OK;
    if (L.count > 0x7FFFFFFFull) return TOOM_EUNSUPPORTED;
    ProfScope ps(down ? CAT_EVAL : CAT_INTERP, st);
    const int cnt = (int)L.count;
    // children and child products: row-major families (child_vec: the
    // level's own buffers, or the staging transposed to the instance-parallel
    // level below)
    const LVec cu = child_vec(plan, l, ws, L.offU, L.e, 0), cv = child_vec(plan, l, ws, L.offV, L.e, 0);
    const LVec cy = child_vec(plan, l, ws, L.offP, 2 * L.e, 0);
    if (cu.ls != 1 || cv.ls != 1 || cy.ls != 1) return TOOM_EUNSUPPORTED;
    if (down) {
        const uint32_t* su = l == 0 ? u : (const uint32_t*)(ws + plan.lv[l - 1].offU);
        const uint32_t* sv = l == 0 ? v : (const uint32_t*)(ws + plan.lv[l - 1].offV);
        const int sgn = (l > 0 || plan.signed_in) ? 1 : 0;
        const int nt = res_threads(L.e);
        const size_t sm = res_eval_smem(L.n);
        dim3 grid((unsigned)cnt, plan.square ? 1 : 2);   // squaring: u only
        uint32_t* du = (uint32_t*)cu.base;
        uint32_t* dv = (uint32_t*)cv.base;
        if (L.B == 3) {
            static bool a = false;
            if (!a) { cudaFuncSetAttribute(k_res_eval<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); a = true; }
            k_res_eval<3><<<grid, nt, sm, st>>>(su, sv, du, dv, cnt, L.n, L.b, L.e, sgn);
        } else {
            static bool a = false;
            if (!a) { cudaFuncSetAttribute(k_res_eval<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); a = true; }
            k_res_eval<4><<<grid, nt, sm, st>>>(su, sv, du, dv, cnt, L.n, L.b, L.e, sgn);
        }
    } else {
        uint32_t* dst = l == 0 ? w : (uint32_t*)(ws + plan.lv[l - 1].offP);
        const int nt = res_threads(L.Lw + 1);   // one round per coefficient row when it fits
        const size_t sm = res_interp_smem(L.B, 2 * L.e, L.Lw, nt);
        const uint32_t* Y = cy.base;
        if (L.B == 3) {
            static bool a = false;
            if (!a) { cudaFuncSetAttribute(k_res_interp<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); a = true; }
            k_res_interp<3><<<cnt, nt, sm, st>>>(Y, dst, 2ll * L.n, cnt, L.n, L.b, 2 * L.e, L.Lw);
        } else {
            static bool a = false;
            if (!a) { cudaFuncSetAttribute(k_res_interp<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); a = true; }
            k_res_interp<4><<<cnt, nt, sm, st>>>(Y, dst, 2ll * L.n, cnt, L.n, L.b, 2 * L.e, L.Lw);
        }
    }
    ps.done(st);
    ++t_launches;
    return TOOM_OK;
}

// ---- lazy levels (csrc/lazy.cuh) ------------------------------------------
// one finishing op: rows of `x` normalised and divided by 2^(32 sa + sr) o
static void lazy_finish(const LzSrc& x, size_t rows, uint32_t* dst, long long dst_is, int Wout, uint32_t o, int shift,
                        LTile* tiles, int cat, cudaStream_t st) {
    if (rows == 0) return;
    ProfScope ps(cat, st);
    constexpr int CH = 16;
    LzFin F;
    F.x = x;
    F.dst = dst;
    F.dst_is = dst_is;
    F.Wout = Wout;
    F.rows = (long long)rows;
    int nt = LV_NT;
    if (Wout <= LV_TL) nt = std::max(32, (int)(((Wout + CH - 1) / CH + 31) / 32 * 32));   // one tile per row
    const int TL = nt * CH;
    F.tpi = (Wout + TL - 1) / TL;
    F.o = o;
    F.oinv = o > 1 ? host_inv32(o) : 1u;
    F.p32 = o > 1 ? host_powmod(2, 32, o) : 0u;
    F.Mch = o > 1 ? host_powmod(2, 32ull * CH, o) : 0u;
    F.mi = o > 1 ? host_invmod(F.Mch, o) : 0u;
    F.sa = shift / 32;
    F.sr = shift % 32;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_lz_fin<CH>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
        attr = true;
    }
    const size_t sm = lz_fin_smem(nt, CH);
    const unsigned grid = (unsigned)(rows * (size_t)F.tpi);
    if (F.tpi == 1) {
        k_lz_fin<CH><<<grid, nt, sm, st>>>(F, tiles, 3);
        ++t_launches;
    } else {
        k_lz_fin<CH><<<grid, nt, sm, st>>>(F, tiles, 1);
        const unsigned long long orcp = o > 1 ? ~0ull / o : 0ull;
        launch_scan2(tiles, (int)rows, F.tpi, 1, nt, &F.o, &orcp, &F.Mch, &F.mi, st);
        k_lz_fin<CH><<<grid, nt, sm, st>>>(F, tiles, 2);
        t_launches += 2;
    }
    ps.done(st);
}

// the level below the lazy block reads interleaved children (fused bottom or a
// staged instance-parallel level) unless it is a long / resident level
static bool lazy_deep_interleaved(const Plan& plan) {
    const size_t nl = (size_t)plan.lz1;
    return nl + 1 >= plan.lv.size() || !plan.lv[nl].lng;
}

static toom_status launch_lazy(const Plan& plan, size_t l, bool down, uint32_t* w, const uint32_t* u, const uint32_t* v,
                               uint8_t* ws, cudaStream_t st) {
    const Level& L = plan.lv[l];
    if (L.count == 0) return TOOM_OK;
    const size_t cc = L.count * (size_t)L.npts;
    LTile* tiles = reinterpret_cast<LTile*>(ws + plan.offLzTiles);
    const bool deepest = (int)l + 1 == plan.lz1;
    const bool il = lazy_deep_interleaved(plan);
    const long long cnt = (long long)L.count;
    if (down) {
        // parents: the user operands (rows), the interleaved lazy children of
        // the lazy level above, or the normalised children of a long level above
        LzSrc pu{}, pv{};
        if (l == 0) {
            pu = LzSrc{u, nullptr, L.n, 1, L.n, plan.signed_in ? 1 : 0};
            pv = LzSrc{v, nullptr, L.n, 1, L.n, plan.signed_in ? 1 : 0};
        } else if (plan.lv[l - 1].lazy) {
            const Level& P = plan.lv[l - 1];
            const size_t half = (size_t)P.e * P.count * P.npts;
            const uint32_t* a = (const uint32_t*)(ws + P.offLzU);
            const uint32_t* b = (const uint32_t*)(ws + P.offLzV);
            pu = LzSrc{a, a + half, 1, cnt, L.n, 0};
            pv = LzSrc{b, b + half, 1, cnt, L.n, 0};
        } else {
            const LVec a = child_vec(plan, l - 1, ws, plan.lv[l - 1].offU, L.n, 0);
            const LVec b = child_vec(plan, l - 1, ws, plan.lv[l - 1].offV, L.n, 0);
            if (a.ls != 1 || b.ls != 1) return TOOM_EUNSUPPORTED;
            pu = LzSrc{a.base, nullptr, L.n, 1, L.n, 1};
            pv = LzSrc{b.base, nullptr, L.n, 1, L.n, 1};
        }
        const unsigned ny = plan.square ? 1 : 2;
        if (deepest && il) {   // evaluation + carry normalisation, interleaved children
            ProfScope ps(CAT_EVAL, st);
            // 64-thread CTAs at 32 registers (launch bounds 64 x 25): all of
            // C4's 2 x 117649 chains resident at once (measured: 128-thread
            // CTAs at 48 registers 327 us, 40 registers without spills 343 us,
            // 32 registers 268 us)
            dim3 grid((unsigned)((L.count + 63) / 64), ny);
            uint32_t* du = (uint32_t*)(ws + L.offU);
            uint32_t* dv = (uint32_t*)(ws + L.offV);
            if (L.B == 3) k_lz_eval_last<3><<<grid, 64, 0, st>>>(pu, pv, du, dv, cnt, L.b, L.lentop, L.e);
            else k_lz_eval_last<4><<<grid, 64, 0, st>>>(pu, pv, du, dv, cnt, L.b, L.lentop, L.e);
            ps.done(st);
            ++t_launches;
            return cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA;
        }
        uint32_t* ul = (uint32_t*)(ws + L.offLzU);
        uint32_t* vl = (uint32_t*)(ws + L.offLzV);
        const size_t half = (size_t)L.e * cc;
        {
            ProfScope ps(CAT_EVAL, st);
            dim3 grid((unsigned)(((size_t)L.e * L.count + 255) / 256), ny);
            const unsigned long long cinv = ~0ull / (unsigned long long)cnt;
            // the first level of a single product: outputs staged, stores in address order
            // (32 -> 16.5 us on C4; with 2B - 1 parents the staged form is no faster: 24 -> 25 us)
            const bool small32 = (unsigned long long)L.e * (unsigned long long)cnt < (1ull << 31) - 256;
            if (small32 && L.B == 4 && cnt == 1) {
                k_lz_eval_small<4, 1><<<grid, 256, 0, st>>>(pu, pv, ul, ul + half, vl, vl + half, L.b, L.lentop, L.e);
            } else if (small32 && L.B == 3 && cnt == 1) {
                k_lz_eval_small<3, 1><<<grid, 256, 0, st>>>(pu, pv, ul, ul + half, vl, vl + half, L.b, L.lentop, L.e);
            } else if (L.B == 3) k_lz_eval<3><<<grid, 256, 0, st>>>(pu, pv, ul, ul + half, vl, vl + half, cnt, cinv, L.b, L.lentop, L.e);
            else k_lz_eval<4><<<grid, 256, 0, st>>>(pu, pv, ul, ul + half, vl, vl + half, cnt, cinv, L.b, L.lentop, L.e);
            ps.done(st);
            ++t_launches;
        }
        if (deepest) {   // row-major normalised children for a long / resident level below
            for (int opd = 0; opd < (plan.square ? 1 : 2); ++opd) {
                const uint32_t* src = opd ? vl : ul;
                const LVec d = child_vec(plan, l, ws, opd ? L.offV : L.offU, L.e, 0);
                if (d.ls != 1) return TOOM_EUNSUPPORTED;
                lazy_finish(LzSrc{src, src + half, 1, (long long)cc, L.e, 0}, cc, (uint32_t*)d.base, L.e, L.e, 1u, 0,
                            tiles, CAT_EVAL, st);
            }
        }
        return cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA;
    }
    // up: the child products, normalised (from below the block) or lazy
    LzSrc y{};
    if (deepest) {
        if (il) {
            y = LzSrc{(const uint32_t*)(ws + L.offP), nullptr, 1, (long long)cc, 2 * L.e, 1};
        } else {
            const LVec a = child_vec(plan, l, ws, L.offP, 2 * L.e, 0);
            if (a.ls != 1) return TOOM_EUNSUPPORTED;
            y = LzSrc{a.base, nullptr, 2 * L.e, 1, 2 * L.e, 1};
        }
    } else {
        const uint32_t* a = (const uint32_t*)(ws + L.offLzP);
        y = LzSrc{a, a + (size_t)L.Wy * cc, 1, (long long)cc, L.Wy, 0};
    }
    // output: interleaved [Wx][count] (the lazy products of the level above)
    uint32_t* xo = (uint32_t*)(ws + ((int)l == plan.lz0 ? plan.offLzX : plan.lv[l - 1].offLzP));
    const size_t xhalf = (size_t)L.Wx * L.count;
    const int MM = (L.Wy + L.b - 1) / L.b;
    {
        ProfScope ps(CAT_INTERP, st);
        const unsigned grid = (unsigned)(((size_t)L.b * L.count + 255) / 256);
        const unsigned long long cinv = ~0ull / (unsigned long long)cnt;
#define TG_LZI(BB, M, Z) k_lz_interp<BB, M, Z><<<grid, 256, 0, st>>>(y, xo, xo + xhalf, cnt, cinv, L.b, L.Wx)
#define TG_LZI2(BB, M) { if (y.hi) TG_LZI(BB, M, true); else TG_LZI(BB, M, false); }
        if (L.B == 3) { if (MM <= 3) TG_LZI2(3, 3) else TG_LZI2(3, 4) }
        else { if (MM <= 3) TG_LZI2(4, 3) else TG_LZI2(4, 4) }
#undef TG_LZI2
#undef TG_LZI
        ps.done(st);
        ++t_launches;
    }
    if ((int)l == plan.lz0) {   // the deferred division, into w or the parent's products
        uint32_t* dst;
        if (l == 0) {
            dst = w;
        } else {
            const LVec d = child_vec(plan, l - 1, ws, plan.lv[l - 1].offP, 2 * L.n, 0);
            if (d.ls != 1) return TOOM_EUNSUPPORTED;
            dst = (uint32_t*)d.base;
        }
        // one finishing division per word factor of the odd part, the shift
        // with the last one; normalised row-major intermediates ping-pong in offLzT
        const size_t nw = plan.lz_o.size();
        LzSrc src{xo, xo + xhalf, 1, cnt, L.Wx, 0};
        uint32_t* tb = (uint32_t*)(ws + plan.offLzT);
        for (size_t i = 0; i < nw; ++i) {
            const bool last = i + 1 == nw;
            uint32_t* d = last ? dst : tb + (i & 1) * (size_t)L.Wx * L.count;
            lazy_finish(src, L.count, d, last ? 2ll * L.n : (long long)L.Wx, last ? 2 * L.n : L.Wx, plan.lz_o[i],
                        last ? plan.lz_s : 0, tiles, CAT_INTERP, st);
            src = LzSrc{d, nullptr, L.Wx, 1, L.Wx, 1};
        }
    }
    return cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA;
}

static toom_status run_plan(const Plan& plan, uint32_t* w, const uint32_t* u, const uint32_t* v, int n, size_t batch,
                            uint8_t* ws, cudaStream_t st) {
    const size_t L = plan.lv.size() - 1;   // number of Toom levels
    toom_status s;
    // long-vector prefix of the recursion
    size_t Tl = 0;
    while (Tl < L && plan.lv[Tl].lng) ++Tl;
    // all ops of the long levels: single-output ops `ops`, multi-output `mops`;
    // launch steps (kind, global index): down in level order, up deepest first
    std::vector<LOpDev> ops;
    std::vector<LMultiDev> mops;
    std::vector<LBigDev> bops;
    std::vector<std::pair<int, int>> sdown, sup;
    LOpDev* ddesc = (LOpDev*)(ws + plan.offDesc);
    LMultiDev* mdesc = (LMultiDev*)(ws + plan.offEDesc);
    LBigDev* bdesc = (LBigDev*)(ws + plan.offBDesc);
    LStatus* status = (LStatus*)(ws + plan.offStatus);
    unsigned* ctr = (unsigned*)(ws + plan.offCtr);
    unsigned epoch = 1;
    auto run_steps = [&](const std::vector<std::pair<int, int>>& steps, int cat) -> toom_status {
        const size_t nops = ops.size();
        for (const auto& stp : steps) {
            toom_status r;
            if (stp.first == 2) {
                r = launch_res(plan, (size_t)stp.second, cat == CAT_EVAL, w, u, v, ws, st);
            } else if (stp.first == 4) {
                r = launch_lazy(plan, (size_t)stp.second, cat == CAT_EVAL, w, u, v, ws, st);
            } else if (stp.first == 3) {
                r = launch_long_big(bops[stp.second], bdesc + stp.second, status, cat, st);
            } else if (stp.first == 0) {
                std::vector<LOpDev> one(1, ops[stp.second]);
                r = launch_long_ops(one, (size_t)stp.second, ddesc, status, ctr, epoch, cat, st);
            } else {
                r = launch_long_multi(mops[stp.second], mdesc + stp.second, status, ctr + nops + stp.second, epoch, cat,
                                      st);
            }
            if (r) return r;
        }
        return TOOM_OK;
    };
    if (Tl) {
        std::vector<std::vector<std::pair<int, int>>> ups(Tl);
        for (size_t l = 0; l < Tl; ++l) {
            if (plan.lv[l].res) {   // instance-resident level: kind 2 steps
                sdown.push_back({2, (int)l});
                ups[l].push_back({2, (int)l});
                continue;
            }
            if (plan.lv[l].lazy) {   // lazy level: kind 4 steps
                sdown.push_back({4, (int)l});
                ups[l].push_back({4, (int)l});
                continue;
            }
            LongCall one;
            build_long_level(plan, l, w, u, v, ws, one);
            const int od = (int)ops.size();
            ops.insert(ops.end(), one.down.begin(), one.down.end());
            const int ou = (int)ops.size();
            ops.insert(ops.end(), one.up.begin(), one.up.end());
            const int md = (int)mops.size();
            mops.insert(mops.end(), one.mdown.begin(), one.mdown.end());
            const int mu = (int)mops.size();
            mops.insert(mops.end(), one.mup.begin(), one.mup.end());
            const int bu = (int)bops.size();
            bops.insert(bops.end(), one.bup.begin(), one.bup.end());
            for (auto x : one.sdown) sdown.push_back({x.first, x.second + (x.first ? md : od)});
            for (auto x : one.sup) ups[l].push_back({x.first, x.second + (x.first == 3 ? bu : (x.first ? mu : ou))});
        }
        for (size_t l = Tl; l-- > 0;) sup.insert(sup.end(), ups[l].begin(), ups[l].end());
        if (lv_build_overflow()) { lv_build_overflow() = false; return TOOM_EUNSUPPORTED; }
        if (ops.size() > plan.nDesc || mops.size() > plan.nDesc || bops.size() > plan.nDesc ||
            ops.size() + mops.size() > plan.nCtr)
            return TOOM_EINVAL;
        if ((s = long_prepare(ops, mops, ddesc, mdesc, status, plan.nStatus, ctr, plan.nCtr, st, &bops, bdesc))) return s;
        if ((s = run_steps(sdown, CAT_EVAL))) return s;
        if (plan.bnd >= 0) {   // row-major children -> interleaved [e][npts*count]
            const Level& Lb = plan.lv[plan.bnd];
            const size_t cc = Lb.count * Lb.npts;
            ProfScope ps(CAT_OTHER, st);
            launch_transpose((const uint32_t*)(ws + plan.offT), (uint32_t*)(ws + Lb.offU), cc, Lb.e, st);
            if (Lb.offV != Lb.offU)   // (squaring: V = U)
                launch_transpose((const uint32_t*)(ws + plan.offT) + cc * Lb.e, (uint32_t*)(ws + Lb.offV), cc, Lb.e, st);
            ps.done(st);
        }
    }
    if (L == 0) {
        // schoolbook only (n <= 64): the base kernel multiplies signed
        // operands, so the unsigned inputs get one zero limb on top
        const int E = n + 1;
        uint32_t* tu = (uint32_t*)ws;
        uint32_t* tv = tu + ((batch * E + 63) & ~(size_t)63);
        uint32_t* tp = tv + ((batch * E + 63) & ~(size_t)63);
        k_transpose_in<<<nblk(batch * E, 256), 256, 0, st>>>(u, tu, batch, n, E, plan.signed_in);
        k_transpose_in<<<nblk(batch * E, 256), 256, 0, st>>>(v, tv, batch, n, E, plan.signed_in);
        if ((s = launch_base(E, tu, tv, tp, batch, st))) return s;
        k_transpose_out<<<nblk(batch * 2 * n, 256), 256, 0, st>>>(tp, w, batch, 2 * n);
        t_launches += 3;
        return TOOM_OK;
    }
    const size_t Lt = plan.fused ? L - 1 : L;   // levels run as staged eval/interp launches
    // down: evaluation
    for (size_t l = Tl; l < Lt; ++l) {
        const Level& Lv = plan.lv[l];
        const uint32_t* su = l == 0 ? u : (const uint32_t*)(ws + plan.lv[l - 1].offU);
        const uint32_t* sv = l == 0 ? v : (const uint32_t*)(ws + plan.lv[l - 1].offV);
        if (l == 0 && top_rows_ok(Lv)) {   // (B = 8 via k_eval_top_rows<8> measured slower: 128 CTAs for C3)
            if ((s = launch_eval_top_rows(Lv, su, sv, (uint32_t*)(ws + Lv.offU), (uint32_t*)(ws + Lv.offV), st, plan.square)))
                return s;
            continue;
        }
        if ((s = launch_eval(Lv.B, l == 0, su, plan.square ? nullptr : sv, (uint32_t*)(ws + Lv.offU),
                             plan.square ? nullptr : (uint32_t*)(ws + Lv.offV), Lv.count, Lv.n,
                             Lv.b, Lv.e, st)))
            return s;
    }
    // bottom
    if (plan.fused) {
        const Level& Lv = plan.lv[L - 1];
        const bool top = (L - 1 == 0);
        const uint32_t* su = top ? u : (const uint32_t*)(ws + plan.lv[L - 2].offU);
        const uint32_t* sv = top ? v : (const uint32_t*)(ws + plan.lv[L - 2].offV);
        uint32_t* out = top ? w : (uint32_t*)(ws + plan.lv[L - 2].offP);
        // a long parent level writes row-major children; a warp-per-product top
        // interpolation reads row-major products
        const int mode = top ? 1 : (plan.lv[L - 2].lazy ? 0 : (plan.lv[L - 2].lng ? 2 : (plan.top_warp ? 3 : 0)));
        if (plan.c2mode == 2) {
            if ((s = launch_fused_dc<4>(Lv, su, sv, out, st))) return s;
        } else if (plan.lzdc) {
            if ((s = launch_fused_dc<3>(Lv, su, sv, out, st))) return s;
        } else if ((s = launch_fused(Lv, mode, su, sv, out, st, plan.square))) {
            return s;
        }
    } else {
        const Level& Lv = plan.lv[L - 1];
        if ((s = launch_base(Lv.e, (const uint32_t*)(ws + Lv.offU), (const uint32_t*)(ws + Lv.offV),
                             (uint32_t*)(ws + Lv.offP), Lv.count * Lv.npts, st)))
            return s;
    }
    // up: interpolation + recomposition
    for (size_t l = Lt; l-- > Tl;) {
        const Level& Lv = plan.lv[l];
        uint32_t* out = l == 0 ? w : (uint32_t*)(ws + plan.lv[l - 1].offP);
        if (l == 0 && plan.top_warp) {
            ProfScope ps(CAT_INTERP, st);
            launch_interp_top_warp(Lv, (const uint32_t*)(ws + Lv.offP), w, st);
            ps.done(st);
            ++t_launches;
            continue;
        }
        if (l == 0 && plan.c2mode) {   // one division over the common denominator (360, or 360^2)
            if ((s = launch_interp_top_cls(Lv, (const uint32_t*)(ws + Lv.offP), w, plan.c2mode == 2, st))) return s;
            continue;
        }
        if (l == 0 && top_rows_ok(Lv) && g_top_stream != 4) {   // mode 4: the per-thread streaming kernel
            if ((s = launch_interp_top_rows(Lv, (const uint32_t*)(ws + Lv.offP), w, st))) return s;
            continue;
        }
        if ((s = launch_interp(Lv.B, l == 0, (const uint32_t*)(ws + Lv.offP), (uint32_t*)(ws + Lv.offW), out, Lv.count,
                               2 * Lv.e, Lv.Lw, Lv.b, 2 * Lv.n, st)))
            return s;
    }
    if (Tl) {
        if (plan.bnd >= 0) {   // interleaved products [2e][npts*count] -> row-major
            const Level& Lb = plan.lv[plan.bnd];
            const size_t cc = Lb.count * Lb.npts;
            ProfScope ps(CAT_OTHER, st);
            launch_transpose((const uint32_t*)(ws + Lb.offP), (uint32_t*)(ws + plan.offT), 2 * Lb.e, cc, st);
            ps.done(st);
        }
        if ((s = run_steps(sup, CAT_INTERP))) return s;
    }
    return TOOM_OK;
}

static bool overlaps(const void* a, size_t an, const void* b, size_t bn) {
    const char* x = (const char*)a;
    const char* y = (const char*)b;
    return x < y + bn && y < x + an;
}

static toom_status check_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) { cudaGetLastError(); return TOOM_ECUDA; }
    return TOOM_OK;
}

static int g_split_streams = [] {
    const char* e = getenv("TOOM_SPLIT_STREAMS");
    return e ? atoi(e) : 1;   // off: two streams measured 1.072 vs 1.075 ms on C2 (no gain), three slower
}();

// device workspace of one call with this plan (the schoolbook-only plan
// needs transposed operand / product buffers instead of level buffers)
static size_t ws_need(const Plan& plan, size_t chunk, size_t n) {
    if (plan.lv.size() == 1) return (2 * ((chunk * (n + 1) + 63) & ~(size_t)63) + 2 * chunk * (n + 1)) * 4;
    return plan.bytes;
}

static toom_status batched(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch,
                           const toom_plan_t& p, cudaStream_t st, bool sgn = false, bool sq = false);

// the batch in g_split_streams parts, each on its own stream with its own
// workspace part, joined back into `st` with events
static toom_status batched_split(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch,
                                 const toom_plan_t& p, cudaStream_t st, bool sgn) {
    const int S = g_split_streams;
    static thread_local std::vector<cudaStream_t> streams;
    static thread_local std::vector<cudaEvent_t> evs;
    if ((int)streams.size() < S) {
        for (int i = (int)streams.size(); i < S; ++i) {
            cudaStream_t x;
            cudaEvent_t e;
            if (cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking) != cudaSuccess) return TOOM_ECUDA;
            cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
            streams.push_back(x);
            evs.push_back(e);
        }
        cudaEvent_t e;
        cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
        evs.push_back(e);
    }
    const size_t part = (batch + S - 1) / S;
    Plan plan;
    toom_status s;
    if ((s = make_plan((int)n, part, p, plan, sgn))) return s;
    const size_t per = (plan.bytes + 255) & ~(size_t)255;
    void* ws = nullptr;
    WsGuard wg;
    if ((s = get_ws(per * S, &ws, st))) return s;
    wg.on = true;
    cudaEvent_t start = evs[S];
    cudaEventRecord(start, st);
    size_t launches = 0;
    for (int i = 0; i < S; ++i) {
        const size_t c0 = (size_t)i * part;
        if (c0 >= batch) break;
        const size_t cnt = std::min(part, batch - c0);
        cudaStreamWaitEvent(streams[i], start, 0);
        Plan pl;
        if ((s = make_plan((int)n, cnt, p, pl, sgn))) return s;
        pl.signed_in = sgn;
        t_launches = 0;
        if ((s = run_plan(pl, w + c0 * 2 * n, u + c0 * n, v + c0 * n, (int)n, cnt, (uint8_t*)ws + (size_t)i * per,
                          streams[i])))
            return s;
        launches += t_launches;
        cudaEventRecord(evs[i], streams[i]);
        cudaStreamWaitEvent(st, evs[i], 0);
    }
    t_launches = launches;
    return cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA;
}

static bool g_verify = false;   // toom_set_verify: residue check of every unsigned result
static bool g_check = false;    // toom_set_check: device exact-division checks

static toom_status batched_core(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch,
                                const toom_plan_t& p, cudaStream_t st, bool sgn, bool sq);

static void launch_verify(const uint32_t* u, size_t nu, const uint32_t* v, size_t nv, const uint32_t* w, size_t batch,
                          cudaStream_t st) {
    if (!batch) return;
    k_verify_m61<<<nblk(batch * 32, 256), 256, 0, st>>>(u, nu, v, nv, w, batch);
    ++t_launches;
}

static toom_status batched(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch,
                           const toom_plan_t& p, cudaStream_t st, bool sgn, bool sq) {
    toom_status s = batched_core(w, u, v, n, batch, p, st, sgn, sq && u == v && !sgn);
    if (s == TOOM_OK && g_verify && !sgn && batch) {
        launch_verify(u, n, v, n, w, batch, st);
        if (cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
    }
    return s;
}

static toom_status batched_core(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch,
                                const toom_plan_t& p, cudaStream_t st, bool sgn, bool sq) {
    t_launches = 0;
    if (n == 0 || n > (1u << 30)) return TOOM_EINVAL;
    if (batch == 0) return TOOM_OK;
    if (!w || !u || !v) return TOOM_EINVAL;
    const size_t in_bytes = n * batch * 4, out_bytes = 2 * n * batch * 4;
    if (overlaps(w, out_bytes, u, in_bytes) || overlaps(w, out_bytes, v, in_bytes)) return TOOM_EINVAL;
    toom_status s = check_device();
    if (s) return s;
    size_t chunk = p.chunk ? p.chunk : batch;
    if (chunk > batch) chunk = batch;
    Plan plan;
    if ((s = make_plan((int)n, chunk, p, plan, sgn, sq))) return s;
    plan.signed_in = sgn;
    if (sgn && plan.lv.size() > 1 && !plan.lv[0].lng) return TOOM_EUNSUPPORTED;   // signed top level: long path only
    // a large batch of short products (no long levels): halves on two streams,
    // so that the kernels of one half (different shared-memory / register
    // shapes) share the SMs with those of the other
    if (!p.chunk && g_split_streams > 1 && batch >= 8192 && !plan.lv[0].lng && !t_prof && plan.lv.size() > 1 && !sq)
        return batched_split(w, u, v, n, batch, p, st, sgn);
    const size_t need = ws_need(plan, chunk, n);
    void* ws = nullptr;
    WsGuard wg;
    if ((s = get_ws(need, &ws, st))) return s;
    wg.on = true;
    for (size_t c0 = 0; c0 < batch; c0 += chunk) {
        const size_t cnt = (batch - c0 < chunk) ? batch - c0 : chunk;
        if (cnt != chunk) {
            Plan p2;
            if ((s = make_plan((int)n, cnt, p, p2, sgn, sq))) return s;
            p2.signed_in = sgn;
            if (sgn && p2.lv.size() > 1 && !p2.lv[0].lng) return TOOM_EUNSUPPORTED;
            if ((s = run_plan(p2, w + c0 * 2 * n, u + c0 * n, v + c0 * n, (int)n, cnt, (uint8_t*)ws, st))) return s;
        } else {
            if ((s = run_plan(plan, w + c0 * 2 * n, u + c0 * n, v + c0 * n, (int)n, cnt, (uint8_t*)ws, st))) return s;
        }
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return TOOM_ECUDA;
    return TOOM_OK;
}

__global__ void k_pad_copy(const uint32_t* __restrict__ src, size_t nsrc, uint32_t* __restrict__ dst, size_t ndst) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < ndst) dst[i] = i < nsrc ? src[i] : 0u;
}

// one top Toom level (count instances of n limbs) run on the long path
static bool long_top_level(size_t n, size_t count, int B, Level& L) {
    LongTables T;
    const PSDesc d = ps_desc(B);
    if (!d.B || !long_tables(B, T) || n > (1u << 30) || !split_ok((int)n, B)) return false;
    L.B = B;
    L.count = count;
    L.n = (int)n;
    L.npts = d.npts;
    L.b = (L.n + B - 1) / B;
    L.lentop = L.n - (B - 1) * L.b;
    L.e = L.b + d.grow;
    L.Lw = 2 * L.b + 1;
    L.lng = true;
    return true;
}

// run long ops with a scratch workspace [slots | status | ctr | desc]; `build`
// appends the ops given the slot pool pointer
template <class BuildF>
static toom_status run_long_standalone(size_t slot_limbs, size_t tiles, size_t nops, BuildF build, cudaStream_t st) {
    auto rnd = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t bS = rnd(slot_limbs * 4), bT = rnd(tiles * sizeof(LStatus)), bC = rnd(nops * 4),
                 bD = rnd(nops * sizeof(LOpDev));
    void* ws = nullptr;
    toom_status s;
    WsGuard wg;
    if ((s = get_ws(bS + bT + bC + bD, &ws, st))) return s;
    wg.on = true;
    uint8_t* base = (uint8_t*)ws;
    LStatus* status = (LStatus*)(base + bS);
    unsigned* ctr = (unsigned*)(base + bS + bT);
    LOpDev* ddesc = (LOpDev*)(base + bS + bT + bC);
    std::vector<LOpDev> ops;
    std::vector<LMultiDev> none;
    build((uint32_t*)base, ops);
    if (lv_build_overflow()) { lv_build_overflow() = false; return TOOM_EUNSUPPORTED; }
    if (ops.size() > nops) return TOOM_EINVAL;
    if ((s = long_prepare(ops, none, ddesc, nullptr, status, tiles, ctr, nops, st))) return s;
    unsigned epoch = 1;
    return launch_long_ops(ops, 0, ddesc, status, ctr, epoch, CAT_OTHER, st);
}

// as run_long_standalone for a whole LongCall (single, multi-output and
// wide-multiplier ops in the call's `sup` order): the stage export of the
// matrix-form Toom-16 interpolation
template <class BuildF>
static toom_status run_long_call_standalone(size_t slot_limbs, size_t tiles, size_t nops, BuildF build, cudaStream_t st) {
    auto rnd = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t bS = rnd(slot_limbs * 4), bT = rnd(tiles * sizeof(LStatus)), bC = rnd(nops * 4),
                 bD = rnd(nops * sizeof(LOpDev)), bM = rnd(nops * sizeof(LMultiDev)), bB = rnd(nops * sizeof(LBigDev));
    void* ws = nullptr;
    toom_status s;
    WsGuard wg;
    if ((s = get_ws(bS + bT + bC + bD + bM + bB, &ws, st))) return s;
    wg.on = true;
    uint8_t* base = (uint8_t*)ws;
    LStatus* status = (LStatus*)(base + bS);
    unsigned* ctr = (unsigned*)(base + bS + bT);
    LOpDev* ddesc = (LOpDev*)(base + bS + bT + bC);
    LMultiDev* mdesc = (LMultiDev*)(base + bS + bT + bC + bD);
    LBigDev* bdesc = (LBigDev*)(base + bS + bT + bC + bD + bM);
    LongCall lc;
    build((uint32_t*)base, lc);
    if (lv_build_overflow()) { lv_build_overflow() = false; return TOOM_EUNSUPPORTED; }
    if (lc.up.size() > nops || lc.mup.size() > nops || lc.bup.size() > nops) return TOOM_EINVAL;
    if ((s = long_prepare(lc.up, lc.mup, ddesc, mdesc, status, tiles, ctr, nops, st, &lc.bup, bdesc))) return s;
    unsigned epoch = 1;
    for (const auto& stp : lc.sup) {
        toom_status r;
        if (stp.first == 3) r = launch_long_big(lc.bup[stp.second], bdesc + stp.second, status, CAT_OTHER, st);
        else if (stp.first == 1) r = launch_long_multi(lc.mup[stp.second], mdesc + stp.second, status, ctr, epoch, CAT_OTHER, st);
        else {
            std::vector<LOpDev> one(1, lc.up[stp.second]);
            r = launch_long_ops(one, (size_t)stp.second, ddesc, status, ctr, epoch, CAT_OTHER, st);
        }
        if (r) return r;
    }
    return TOOM_OK;
}

// ---- NTT inner multiplier (ntt.cuh) ----------------------
struct NttTables {
    int N = 0;
    uint64_t* tw = nullptr;    // omega^k, k < N/2
    uint64_t* twi = nullptr;   // omega^-k
    uint64_t ninv = 0;
};
static std::mutex g_ntt_mu;
static std::vector<NttTables> g_ntt_tables;

static toom_status ntt_tables(int N, NttTables& out) {
    std::lock_guard<std::mutex> g(g_ntt_mu);
    for (auto& t : g_ntt_tables)
        if (t.N == N) { out = t; return TOOM_OK; }
    NttTables t;
    t.N = N;
    const uint64_t w = gl_pow(NTT_G, (NTT_P - 1) / (uint64_t)N), wi = gl_pow(w, NTT_P - 2);
    std::vector<uint64_t> h((size_t)N / 2), hi((size_t)N / 2);
    uint64_t x = 1, y = 1;
    for (int k = 0; k < N / 2; ++k) { h[k] = x; hi[k] = y; x = gl_mul(x, w); y = gl_mul(y, wi); }
    if (cudaMalloc(&t.tw, (size_t)N / 2 * 8) != cudaSuccess || cudaMalloc(&t.twi, (size_t)N / 2 * 8) != cudaSuccess) {
        cudaGetLastError();
        return TOOM_ENOMEM;
    }
    cudaMemcpy(t.tw, h.data(), (size_t)N / 2 * 8, cudaMemcpyHostToDevice);
    cudaMemcpy(t.twi, hi.data(), (size_t)N / 2 * 8, cudaMemcpyHostToDevice);
    t.ninv = gl_pow((uint64_t)N, NTT_P - 2);
    g_ntt_tables.push_back(t);
    out = t;
    return TOOM_OK;
}

static int ntt_size(int e) {
    int N = NTT_SB;
    while (N < 4 * e) N <<= 1;
    return N;
}
// workspace of ntt_products: digit arrays A, B ([count][N] u64), lowest-nonzero
// indices, the carry op's tile records / counters / descriptor
static size_t ntt_ws_bytes(int e, int count) {
    const size_t N = (size_t)ntt_size(e);
    const size_t tiles = long_tiles((size_t)count, 2 * e);
    return 2 * N * count * 8 + 3 * 256 + (size_t)count * 16 + tiles * sizeof(LStatus) + 256 + sizeof(LOpDev) + 1024;
}

// Y[c] = U[c] * V[c] (two's complement, e limbs each -> 2e limbs) for c < count,
// through the exact NTT over p = 2^64 - 2^32 + 1 (magnitudes, sign applied)
static toom_status ntt_products(uint32_t* Y, long long y_is, const uint32_t* U, long long u_is, const uint32_t* V,
                                long long v_is, int e, int count, uint8_t* ws, cudaStream_t st, bool sgn = true) {
    if (count == 0) return TOOM_OK;
    const int N = ntt_size(e);
    NttTables T;
    toom_status s;
    if ((s = ntt_tables(N, T))) return s;
    auto rnd = [](size_t b) { return (b + 255) & ~(size_t)255; };
    uint64_t* A = (uint64_t*)ws;
    uint64_t* Bv = A + (size_t)N * count;
    uint8_t* p = ws + 2 * (size_t)N * count * 8;
    int* zu = (int*)p;
    int* zv = zu + count;
    int* zw = zv + count;
    p += rnd((size_t)count * 12);
    LStatus* status = (LStatus*)p;
    const size_t tiles = long_tiles((size_t)count, 2 * e);
    p += rnd(tiles * sizeof(LStatus));
    unsigned* ctr = (unsigned*)p;
    p += 256;
    LOpDev* desc = (LOpDev*)p;
    cudaMemsetAsync(zu, 0x7F, (size_t)count * 12, st);
    const dim3 gz((unsigned)std::min(64, (e + 255) / 256), (unsigned)count);
    k_ntt_lowest_nz<<<gz, 256, 0, st>>>(U, u_is, e, zu);
    k_ntt_lowest_nz<<<gz, 256, 0, st>>>(V, v_is, e, zv);
    const dim3 gd((unsigned)std::min(1024, N / 256), (unsigned)count);
    k_ntt_digits<<<gd, 256, 0, st>>>(U, u_is, e, sgn ? 1 : 0, zu, A, N);
    k_ntt_digits<<<gd, 256, 0, st>>>(V, v_is, e, sgn ? 1 : 0, zv, Bv, N);
    t_launches += 4;
    const dim3 gs((unsigned)std::min(2048, N / 2 / 256), (unsigned)count), gt((unsigned)(N / NTT_SB), (unsigned)count);
    const dim3 g8((unsigned)std::min(2048, std::max(1, N / 8 / 256)), (unsigned)count);
    for (uint64_t* X : {A, Bv}) {
        // global stages three at a time (radix 8), the rest radix 2, then the
        // stages below NTT_SB in shared memory
        int h = N / 2;
        for (; h / 4 >= NTT_SB; h /= 8) { k_ntt_r8<false><<<g8, 256, 0, st>>>(X, N, h / 4, T.tw); ++t_launches; }
        for (; h >= NTT_SB; h >>= 1) { k_ntt_dif_stage<<<gs, 256, 0, st>>>(X, N, h, T.tw); ++t_launches; }
        k_ntt_dif_tail<<<gt, 512, 0, st>>>(X, N, T.tw);
        ++t_launches;
    }
    k_ntt_pointwise<<<2048, 256, 0, st>>>(A, Bv, (long long)N * count, T.ninv);
    k_ntt_dit_head<<<gt, 512, 0, st>>>(A, N, T.twi);
    t_launches += 2;
    {
        int h = NTT_SB;
        const int nglob = [&] { int k = 0; for (int x = NTT_SB; x < N; x <<= 1) ++k; return k; }();
        for (int r = 0; r < nglob % 3; ++r, h <<= 1) { k_ntt_dit_stage<<<gs, 256, 0, st>>>(A, N, h, T.twi); ++t_launches; }
        for (; h < N; h <<= 3) { k_ntt_r8<true><<<g8, 256, 0, st>>>(A, N, h, T.twi); ++t_launches; }
    }
    // w = sum_k c_k 2^(16 k), c_k = lo_k + hi_k 2^32 < 2^53: four strided word
    // slices of the coefficient array (lo/hi of the even / odd digits)
    {
        const uint32_t* X = (const uint32_t*)A;
        LOpBuilder b(Y, y_is, 1, 2 * e, count);
        const long long is = 2ll * N;
        b.add(LVec{X + 0, is, 4, N / 2, 0}, 1, 0);
        b.add(LVec{X + 2, is, 4, N / 2, 0}, 1, 16);
        b.add(LVec{X + 1, is, 4, N / 2, 0}, 1, 32);
        b.add(LVec{X + 3, is, 4, N / 2, 0}, 1, 48);
        b.op.wide = 0;
        std::vector<LOpDev> ops(1, b.op);
        std::vector<LMultiDev> none;
        if ((s = long_prepare(ops, none, desc, nullptr, status, tiles, ctr, 1, st))) return s;
        unsigned epoch = 1;
        if ((s = launch_long_ops(ops, 0, desc, status, ctr, epoch, CAT_BASE, st))) return s;
    }
    // the sign: negate the products of operands of different signs
    const dim3 gw((unsigned)std::min(64, (2 * e + 255) / 256), (unsigned)count);
    if (sgn) {
        k_ntt_lowest_nz<<<gw, 256, 0, st>>>(Y, y_is, 2 * e, zw);
        k_ntt_negate<<<gw, 256, 0, st>>>(Y, y_is, 2 * e, U, u_is, e, V, v_is, e, zw);
        t_launches += 2;
    }
    return cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA;
}

}  // namespace tg

using namespace tg;

extern "C" {

toom_status toom_mul_signed_batched(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch,
                                    const toom_plan_t* plan, void* stream) {
    if (!plan) return fail(TOOM_EINVAL);
    return fail(batched(w, u, v, n, batch, *plan, (cudaStream_t)stream, true));
}

toom_status toom_eval_points(uint32_t* out, const uint32_t* a, size_t n, size_t batch, int B, int is_signed,
                             void* stream) {
    t_launches = 0;
    Level L;
    if (!out || !a || !long_top_level(n, batch, B, L)) return fail(TOOM_EINVAL);
    if (batch == 0) return TOOM_OK;
    if (overlaps(out, (size_t)L.npts * batch * L.e * 4, a, n * batch * 4)) return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    LongTables T;
    long_tables(B, T);
    const LVec par{a, (long long)n, 1, (int)n, is_signed ? 1 : 0};
    s = run_long_standalone(0, long_tiles(batch, L.e), (size_t)T.neo,
                            [&](uint32_t*, std::vector<LOpDev>& ops) {
                                long_eval_ops(L, par, [&](int k) { return LVec{out + (size_t)k * batch * L.e, L.e, 1, L.e, 1}; }, ops);
                            },
                            (cudaStream_t)stream);
    if (s == TOOM_OK && cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
    return fail(s);
}

toom_status toom_eval_points_range(uint32_t* out, const uint32_t* a, size_t n, size_t batch, int B, int is_signed,
                                   int k0, int k1, void* stream) {
    t_launches = 0;
    Level L;
    if (!a || !long_top_level(n, batch, B, L) || k0 < 0 || k1 > L.npts || k0 > k1) return fail(TOOM_EINVAL);
    if (batch == 0 || k0 == k1) return TOOM_OK;   // (an empty range: out may be null)
    if (!out) return fail(TOOM_EINVAL);
    if (overlaps(out, (size_t)(k1 - k0) * batch * L.e * 4, a, n * batch * 4)) return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    LongTables T;
    long_tables(B, T);
    // every evaluation op writes one point (the programs' eval ops are one per point)
    for (int k = 0; k < T.neo; ++k)
        if (T.eo[k].dst < 0 || T.eo[k].dst >= L.npts) return fail(TOOM_EUNSUPPORTED);
    const LVec par{a, (long long)n, 1, (int)n, is_signed ? 1 : 0};
    s = run_long_standalone(0, long_tiles(batch, L.e), (size_t)T.neo,
                            [&](uint32_t*, std::vector<LOpDev>& ops) {
                                long_eval_ops(L, par, [&](int k) { return LVec{out + (size_t)k * batch * L.e, L.e, 1, L.e, 1}; },
                                              ops, k0, k1);
                            },
                            (cudaStream_t)stream);
    if (s == TOOM_OK && cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
    return fail(s);
}

toom_status toom_interp_recompose(uint32_t* w, const uint32_t* y, size_t n, size_t batch, int B, void* stream) {
    t_launches = 0;
    Level L;
    if (!w || !y || !long_top_level(n, batch, B, L)) return fail(TOOM_EINVAL);
    if (batch == 0) return TOOM_OK;
    if (overlaps(w, 2 * n * batch * 4, y, (size_t)L.npts * batch * 2 * L.e * 4)) return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    LongTables T;
    long_tables(B, T);
    const int Wt = long_Wt(L);
    const size_t slot_limbs = (size_t)long_nslots(B, T.nslots) * batch * Wt;
    if (B == 16 && g_t16_matrix) {   // the matrix form (f1)
        s = run_long_call_standalone(slot_limbs, long_tiles(batch, std::max(Wt, 2 * L.n)) * (size_t)L.npts, 64,
                                     [&](uint32_t* slots, LongCall& lc) {
                                         long_t16_matrix(L, [&](int k) { return LVec{y + (size_t)k * batch * 2 * L.e, 2 * L.e, 1, 2 * L.e, 1}; },
                                                         slots, w, lc);
                                     },
                                     (cudaStream_t)stream);
        if (s == TOOM_OK && cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
        return fail(s);
    }
    s = run_long_standalone(slot_limbs, long_tiles(batch, std::max(Wt, 2 * L.n)), (size_t)T.nio + 1,
                            [&](uint32_t* slots, std::vector<LOpDev>& ops) {
                                long_interp_ops(L, [&](int k) { return LVec{y + (size_t)k * batch * 2 * L.e, 2 * L.e, 1, 2 * L.e, 1}; },
                                                slots, w, ops);
                            },
                            (cudaStream_t)stream);
    if (s == TOOM_OK && cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
    return fail(s);
}

toom_status toom_mul_ntt(uint32_t* w, const uint32_t* u, size_t nu, const uint32_t* v, size_t nv, int B, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    t_launches = 0;
    if (!w || !u || !v || nu == 0 || nv == 0 || nu > (1u << 28) || nv > (1u << 28)) return fail(TOOM_EINVAL);
    if (overlaps(w, (nu + nv) * 4, u, nu * 4) || overlaps(w, (nu + nv) * 4, v, nv * 4)) return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    const size_t n = std::max(nu, nv);
    auto rnd = [](size_t b) { return (b + 255) & ~(size_t)255; };
    if (B == 0) {   // the inner multiplier alone: one product of n-limb (zero-padded) operands
        const size_t e = n;       // unsigned operands (no sign handling)
        const size_t bU = rnd(e * 4), bY = rnd(2 * e * 4), bN = rnd(ntt_ws_bytes((int)e, 1));
        void* ws = nullptr;
        WsGuard wg;
        if ((s = get_ws(2 * bU + bY + bN, &ws, st))) return fail(s);
        wg.on = true;
        uint32_t* pu = (uint32_t*)ws;
        uint32_t* pv = (uint32_t*)((uint8_t*)ws + bU);
        uint32_t* py = (uint32_t*)((uint8_t*)ws + 2 * bU);
        k_pad_copy<<<nblk(e, 256), 256, 0, st>>>(u, nu, pu, e);
        k_pad_copy<<<nblk(e, 256), 256, 0, st>>>(v, nv, pv, e);
        if ((s = ntt_products(py, 2 * e, pu, e, pv, e, (int)e, 1, (uint8_t*)ws + 2 * bU + bY, st, false))) return fail(s);
        k_pad_copy<<<nblk(nu + nv, 256), 256, 0, st>>>(py, nu + nv, w, nu + nv);
        t_launches += 3;
        return fail(cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA);
    }
    // Toom-B top level on the long-vector kernels, its 2B-1 products by the NTT
    Level L;
    if (!long_top_level(n, 1, B, L)) return fail(TOOM_EINVAL);
    const size_t np = (size_t)L.npts, e = (size_t)L.e;
    LongTables T;
    long_tables(B, T);
    const int Wt = long_Wt(L);
    // scratch of the stage calls (the larger of evaluation and interpolation)
    const size_t stage = rnd((size_t)long_nslots(B, T.nslots) * Wt * 4) +
                         rnd(long_tiles(1, std::max(Wt, 2 * L.n)) * (size_t)L.npts * sizeof(LStatus)) +
                         rnd(4096 * 4) + rnd(4096 * sizeof(LOpDev)) + rnd(64 * sizeof(LMultiDev)) +
                         rnd(64 * sizeof(LBigDev)) + (1 << 20);
    const size_t bP = rnd(n * 4), bE = rnd(np * e * 4), bY = rnd(np * 2 * e * 4), bN = rnd(ntt_ws_bytes((int)e, (int)np));
    void* ws = nullptr;
    WsGuard wg;
    if ((s = get_ws(2 * bP + 2 * bE + bY + std::max(bN, stage) + rnd(2 * n * 4), &ws, st))) return fail(s);
    wg.on = true;
    uint8_t* p = (uint8_t*)ws;
    uint32_t* pu = (uint32_t*)p; p += bP;
    uint32_t* pv = (uint32_t*)p; p += bP;
    uint32_t* EU = (uint32_t*)p; p += bE;
    uint32_t* EV = (uint32_t*)p; p += bE;
    uint32_t* Yp = (uint32_t*)p; p += bY;
    uint32_t* pw = (uint32_t*)p; p += rnd(2 * n * 4);
    uint8_t* scratch = p;
    k_pad_copy<<<nblk(n, 256), 256, 0, st>>>(u, nu, pu, n);
    k_pad_copy<<<nblk(n, 256), 256, 0, st>>>(v, nv, pv, n);
    size_t launches = 2;
    // the stage exports run with the scratch region as their workspace
    t_ws_override = scratch;
    t_ws_override_bytes = std::max(bN, stage);
    s = toom_eval_points(EU, pu, n, 1, B, 0, stream);
    launches += t_launches;
    if (!s) { s = toom_eval_points(EV, pv, n, 1, B, 0, stream); launches += t_launches; }
    t_launches = 0;
    if (!s) s = ntt_products(Yp, 2 * e, EU, e, EV, e, (int)e, (int)np, scratch, st);
    launches += t_launches;
    if (!s) { s = toom_interp_recompose(pw, Yp, n, 1, B, stream); launches += t_launches; }
    t_ws_override = nullptr;
    t_ws_override_bytes = 0;
    if (s) return fail(s);
    k_pad_copy<<<nblk(nu + nv, 256), 256, 0, st>>>(pw, nu + nv, w, nu + nv);
    t_launches = launches + 1;
    if (g_verify) launch_verify(u, nu, v, nv, w, 1, st);
    return fail(cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA);
}

toom_plan_t toom_default_plan(int B) {
    toom_plan_t p;
    p.top_B = B;
    p.t4 = 256;
    p.t3 = 64;
    p.chunk = 0;
    p.long_count = 0;
    return p;
}

toom_status toom_mul_batched_plan(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch,
                                  const toom_plan_t* plan, void* stream) {
    if (!plan) return fail(TOOM_EINVAL);
    return fail(batched(w, u, v, n, batch, *plan, (cudaStream_t)stream));
}

toom_status toom_mul_batched(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t n, size_t batch, int B,
                             void* stream) {
    if (B != 3 && B != 4 && B != 8 && B != 16 && B != 32) return fail(TOOM_EINVAL);
    toom_plan_t p = toom_default_plan(B);
    return fail(batched(w, u, v, n, batch, p, (cudaStream_t)stream));
}

toom_status toom_sqr_batched(uint32_t* w, const uint32_t* u, size_t n, size_t batch, const toom_plan_t* plan,
                             void* stream) {
    if (!plan) return fail(TOOM_EINVAL);
    return fail(batched(w, u, u, n, batch, *plan, (cudaStream_t)stream, false, true));
}

toom_status toom_mul(uint32_t* w, const uint32_t* u, size_t nu, const uint32_t* v, size_t nv, int B, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    t_launches = 0;
    if (!w || (nu && !u) || (nv && !v)) return fail(TOOM_EINVAL);
    if (B != 3 && B != 4 && B != 8 && B != 16 && B != 32) return fail(TOOM_EINVAL);
    if ((nu && overlaps(w, (nu + nv) * 4, u, nu * 4)) || (nv && overlaps(w, (nu + nv) * 4, v, nv * 4)))
        return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    if (nu == 0 || nv == 0) {
        if (nu + nv) cudaMemsetAsync(w, 0, (nu + nv) * 4, st);
        return fail(cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA);
    }
    const size_t n = nu > nv ? nu : nv;
    toom_plan_t p = toom_default_plan(B);
    if (nu == nv) return fail(batched(w, u, v, n, 1, p, st, false, u == v));   // w has 2n limbs: no copies; u == v squares
    // unbalanced: the shorter operand zero-padded to n limbs in
    // the call's workspace, behind the plan's own scratch; w has nu+nv < 2n
    // limbs, so the 2n-limb product also lives in the workspace and its low
    // nu+nv limbs (the high ones are zero) are copied out
    Plan pl;
    if ((s = make_plan((int)n, 1, p, pl))) return fail(s);
    const size_t wsb = (ws_need(pl, 1, n) + 255) & ~(size_t)255;
    const size_t pad = ((4 * n * 4) + 255) & ~(size_t)255;
    void* ws = nullptr;
    WsGuard wg;
    if ((s = get_ws(wsb + pad, &ws, st))) return fail(s);
    wg.on = true;
    uint32_t* pu = (uint32_t*)((uint8_t*)ws + wsb);
    uint32_t* pv = pu + n;
    uint32_t* pw = pv + n;
    const uint32_t* su = u;
    const uint32_t* sv = v;
    if (nu < n) { k_pad_copy<<<nblk(n, 256), 256, 0, st>>>(u, nu, pu, n); su = pu; }
    if (nv < n) { k_pad_copy<<<nblk(n, 256), 256, 0, st>>>(v, nv, pv, n); sv = pv; }
    t_ws_override = ws;
    t_ws_override_bytes = wsb;
    s = batched(pw, su, sv, n, 1, p, st);
    t_ws_override = nullptr;
    t_ws_override_bytes = 0;
    if (s == TOOM_OK) {
        k_pad_copy<<<nblk(nu + nv, 256), 256, 0, st>>>(pw, nu + nv, w, nu + nv);
        t_launches += 2;
    }
    if (s == TOOM_OK && cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
    return fail(s);
}

toom_status toom_mul_batched_host(uint32_t* w_host, const uint32_t* u_host, const uint32_t* v_host, size_t n,
                                  size_t batch, const toom_plan_t* plan, void* stream) {
    cudaStream_t st = (cudaStream_t)stream;
    if (!w_host || !u_host || !v_host || !plan || n == 0) return fail(TOOM_EINVAL);
    if (batch == 0) return TOOM_OK;
    toom_status s = check_device();
    if (s) return fail(s);
    // Pipeline: K chunks round-robin over NS streams, each chunk H2D(u, v) ->
    // multiply (own workspace) -> D2H(w) in its stream's order, so the copies
    // of one chunk overlap the kernels of another (pinned host buffers overlap;
    // pageable ones still give the right result).
    constexpr int NS = 3;
    static const int kmax = [] {
        const char* e = getenv("TOOM_HOST_CHUNKS");
        return e ? atoi(e) : 8;
    }();
    const int K = batch >= 4096 ? (int)std::min<size_t>((size_t)kmax, batch / 512) : 1;
    const size_t chunk = (batch + K - 1) / K;
    static std::mutex mu;
    static uint8_t* dbuf = nullptr;
    static size_t dbytes = 0;
    static cudaStream_t ss[NS];
    static cudaEvent_t ev[NS + 1];
    static bool init = false;
    std::lock_guard<std::mutex> g(mu);
    if (!init) {
        for (int i = 0; i < NS; ++i) {
            if (cudaStreamCreateWithFlags(&ss[i], cudaStreamNonBlocking) != cudaSuccess) return fail(TOOM_ECUDA);
            cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
        }
        cudaEventCreateWithFlags(&ev[NS], cudaEventDisableTiming);
        init = true;
    }
    toom_plan_t pc = *plan;
    pc.chunk = 0;
    Plan pl;
    if ((s = make_plan((int)n, chunk, pc, pl))) return fail(s);
    size_t wsb = ws_need(pl, chunk, n);
    wsb = (wsb + 255) & ~(size_t)255;
    const size_t io = ((4 * n * chunk * 4) + 255) & ~(size_t)255;   // u, v, w of a chunk
    const size_t per = io + wsb;
    const int nslot = std::min(NS, K);
    if (per * nslot > dbytes) {
        if (dbuf) { cudaDeviceSynchronize(); cudaFree(dbuf); dbuf = nullptr; dbytes = 0; }
        if (cudaMalloc((void**)&dbuf, per * nslot) != cudaSuccess) { cudaGetLastError(); return fail(TOOM_ENOMEM); }
        dbytes = per * nslot;
    }
    cudaEventRecord(ev[NS], st);
    for (int i = 0; i < nslot; ++i) cudaStreamWaitEvent(ss[i], ev[NS], 0);
    size_t launches = 0;
    for (int i = 0; i < K; ++i) {
        const size_t c0 = (size_t)i * chunk;
        if (c0 >= batch) break;
        const size_t cnt = std::min(chunk, batch - c0);
        const int sl = i % nslot;
        cudaStream_t cs = ss[sl];
        uint8_t* base = dbuf + (size_t)sl * per;
        uint32_t* du = (uint32_t*)base;
        uint32_t* dv = du + n * cnt;
        uint32_t* dw = dv + n * cnt;
        if (cudaMemcpyAsync(du, u_host + c0 * n, n * cnt * 4, cudaMemcpyHostToDevice, cs) != cudaSuccess ||
            cudaMemcpyAsync(dv, v_host + c0 * n, n * cnt * 4, cudaMemcpyHostToDevice, cs) != cudaSuccess)
            return fail(TOOM_ECUDA);
        t_ws_override = base + io;
        t_ws_override_bytes = wsb;
        s = batched(dw, du, dv, n, cnt, pc, cs);
        t_ws_override = nullptr;
        t_ws_override_bytes = 0;
        if (s) return fail(s);
        launches += t_launches;
        if (cudaMemcpyAsync(w_host + c0 * 2 * n, dw, 2 * n * cnt * 4, cudaMemcpyDeviceToHost, cs) != cudaSuccess)
            return fail(TOOM_ECUDA);
    }
    for (int i = 0; i < nslot; ++i) {
        cudaEventRecord(ev[i], ss[i]);
        cudaStreamWaitEvent(st, ev[i], 0);
    }
    t_launches = launches;
    if (cudaStreamSynchronize(st) != cudaSuccess) return fail(TOOM_ECUDA);
    return TOOM_OK;
}

size_t toom_workspace_bytes(size_t n, size_t batch, const toom_plan_t* plan) {
    if (!plan || n == 0) return 0;
    toom_plan_t p = *plan;
    size_t chunk = p.chunk ? p.chunk : batch;
    if (chunk > batch) chunk = batch;
    Plan pl;
    if (make_plan((int)n, chunk, p, pl) != TOOM_OK) return 0;
    return ws_need(pl, chunk, n);
}

toom_status toom_set_workspace(void* dev_ptr, size_t bytes) {
    std::lock_guard<std::mutex> g(g_ws_mu);
    std::lock_guard<std::mutex> gu(g_user_mu);   // no call is using the caller buffer
    // the library's own buffers are released (after the device drained)
    if (!g_ws_list.empty()) cudaDeviceSynchronize();
    for (auto& e : g_ws_list) cudaFree(e.p);
    g_ws_list.clear();
    if (g_user_ws && g_user_used) cudaEventSynchronize(g_user_ev);   // the previous caller buffer is idle
    g_user_ws = dev_ptr;
    g_user_bytes = dev_ptr ? bytes : 0;
    g_user_used = false;
    g_user_last = nullptr;
    return TOOM_OK;
}

toom_status toom_last_error(void) {
    toom_status s = t_last;
    t_last = TOOM_OK;
    if (g_check || g_verify) {
        // device-detected failures: read back and clear
        unsigned f = 0;
        if (cudaDeviceSynchronize() != cudaSuccess || cudaMemcpyFromSymbol(&f, tg_err_flags, sizeof f) != cudaSuccess) {
            cudaGetLastError();
            return s == TOOM_OK ? TOOM_ECUDA : s;
        }
        if (f) {
            const unsigned z = 0;
            cudaMemcpyToSymbol(tg_err_flags, &z, sizeof z);
            if (s == TOOM_OK) s = (f & 1u) ? TOOM_EINEXACT : TOOM_EVERIFY;
        }
    }
    return s;
}

void toom_set_check(int on) {
    g_check = on != 0;
    const int v = g_check ? 1 : 0;
    cudaMemcpyToSymbol(tg_check_on, &v, sizeof v);
    cudaGetLastError();
}

void toom_set_verify(int on) { g_verify = on != 0; }

void toom_debug_fault(int kind) {
    const int v = kind;
    cudaMemcpyToSymbol(tg_fault, &v, sizeof v);
    cudaGetLastError();
}

const char* toom_status_string(toom_status s) {
    switch (s) {
        case TOOM_OK: return "TOOM_OK";
        case TOOM_EINVAL: return "TOOM_EINVAL";
        case TOOM_EVERIFY: return "TOOM_EVERIFY";
        case TOOM_EINEXACT: return "TOOM_EINEXACT";
        case TOOM_ENOMEM: return "TOOM_ENOMEM";
        case TOOM_ECUDA: return "TOOM_ECUDA";
        case TOOM_EUNSUPPORTED: return "TOOM_EUNSUPPORTED";
    }
    return "unknown";
}

size_t toom_last_launch_count(void) { return t_launches; }

toom_status toom_base_interleaved(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t E, size_t count,
                                  void* stream) {
    t_launches = 0;
    if (!w || !u || !v || E < 1 || E > 64) return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    s = launch_base((int)E, u, v, w, count, (cudaStream_t)stream);
    if (s == TOOM_OK && cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
    return fail(s);
}

// the base case on the int8 tensor cores (csrc/tc_base.cuh)
toom_status toom_base_interleaved_tc(uint32_t* w, const uint32_t* u, const uint32_t* v, size_t E, size_t count,
                                     void* stream) {
    t_launches = 0;
    if (!w || !u || !v || E < 1) return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    if (count == 0) return TOOM_OK;
    const cudaStream_t st = (cudaStream_t)stream;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = (unsigned)std::min<size_t>(count, (size_t)sms * 8);
    ProfScope ps(CAT_BASE, st);
    switch (E) {
#define TG_TCB(EE) case EE: k_base_tc<EE><<<grid, 128, 0, st>>>(u, v, w, count); break;
        TG_TCB(2) TG_TCB(5) TG_TCB(9) TG_TCB(16) TG_TCB(17) TG_TCB(18) TG_TCB(23) TG_TCB(24)
#undef TG_TCB
        default: return fail(TOOM_EUNSUPPORTED);
    }
    ps.done(st);
    ++t_launches;
    s = cudaGetLastError() == cudaSuccess ? TOOM_OK : TOOM_ECUDA;
    return fail(s);
}

int toom_npoints(int B) { return ps_desc(B).npts; }

void toom_set_top_stream(int on) { g_top_stream = on; }

void toom_set_t16_matrix(int on) { g_t16_matrix = on != 0; }
void toom_set_c2_mode(int mode) { g_c2mode = (mode >= 0 && mode <= 2) ? mode : 0; }
void toom_set_lazy_bottom(int on) { g_lzdc = on != 0; }

void toom_set_fused(int on) {
    // 0: every level staged (k_eval / k_base / k_interp); 1: fused bottom level
    // and warp-per-row top level (default)
    g_disable_fused = (on == 0);
    g_disable_toprows = (on == 0);
}

void toom_profile_enable(int on) {
    t_prof = on != 0;
}

int toom_profile_collect(double* ms, size_t* launches, int ncat) {
    for (int c = 0; c < ncat; ++c) { ms[c] = 0; launches[c] = 0; }
    if (t_prof_stream || !t_prof_recs.empty()) cudaDeviceSynchronize();
    for (auto& r : t_prof_recs) {
        float t = 0;
        cudaEventElapsedTime(&t, r.a, r.b);
        if (r.cat < ncat) { ms[r.cat] += t; launches[r.cat] += 1; }
        t_prof_pool.push_back(r.a);
        t_prof_pool.push_back(r.b);
    }
    t_prof_recs.clear();
    return NCAT;
}

size_t toom_plan_describe(size_t n, size_t batch, const toom_plan_t* plan, char* buf, size_t len) {
    if (!plan || n == 0) return 0;
    Plan pl;
    toom_plan_t p = *plan;
    if (make_plan((int)n, batch, p, pl) != TOOM_OK) return 0;
    std::string js = "{\"levels\": [";
    for (size_t l = 0; l < pl.lv.size(); ++l) {
        const Level& L = pl.lv[l];
        char tmp[512];
        snprintf(tmp, sizeof tmp,
                 "%s{\"B\": %d, \"count\": %zu, \"n\": %d, \"b\": %d, \"lentop\": %d, \"e\": %d, \"Lw\": %d, \"npts\": %d, \"long\": %s, \"res\": %s, \"lazy\": %s}",
                 l ? ", " : "", L.B, L.count, L.n, L.b, L.lentop, L.e, L.Lw, L.npts, L.lng ? "true" : "false",
                 L.res ? "true" : "false", L.lazy ? "true" : "false");
        js += tmp;
    }
    char tail[128];
    snprintf(tail, sizeof tail,
             "], \"workspace_bytes\": %zu, \"fused_bottom\": %s, \"c2_mode\": %d, \"lazy_bottom_dc\": %s}", pl.bytes,
             pl.fused ? "true" : "false", pl.c2mode, pl.lzdc ? "true" : "false");
    js += tail;
    if (buf && len) {
        size_t k = js.size() < len - 1 ? js.size() : len - 1;
        memcpy(buf, js.data(), k);
        buf[k] = 0;
    }
    return js.size() + 1;
}

size_t toom_product_width_point(size_t n, int B) { return 2 * toom_eval_width(n, B); }

size_t toom_eval_width(size_t n, int B) {
    const PSDesc d = ps_desc(B);
    if (!d.B || n == 0) return 0;
    const size_t b = (n + B - 1) / B;
    return b + d.grow;
}

toom_status toom_eval_top(uint32_t* out, const uint32_t* a, size_t n, size_t batch, int B, void* stream) {
    t_launches = 0;
    const PSDesc d = ps_desc(B);
    if (!out || !a || !d.B || n < (size_t)(2 * B)) return fail(TOOM_EINVAL);
    const int b = (int)((n + B - 1) / B);
    if ((int)n - (B - 1) * b < 1) return fail(TOOM_EINVAL);
    toom_status s = check_device();
    if (s) return fail(s);
    const int e = (int)toom_eval_width(n, B);
    // the two-operand kernel with no second operand (srcV = nullptr: one
    // thread per instance, every output limb stored once)
    s = launch_eval(B, true, a, nullptr, out, nullptr, batch, (int)n, b, e, (cudaStream_t)stream);
    if (s == TOOM_OK && cudaGetLastError() != cudaSuccess) s = TOOM_ECUDA;
    return fail(s);
}

}  // extern "C"
