// Top-level evaluation (step a1+a2) and interpolation + recomposition
// (steps a4+a5) for batched products whose top level is Toom-3/Toom-4, with
// one warp per point / per coefficient row and one lane per product.
//
//   k_eval_top_rows<B>    CTA = 32 products x NP warps.  Row-major operand
//                         limbs are staged through smem in chunks of CH limbs
//                         with coalesced loads; warp k streams U(x_k), V(x_k)
//                         (homogeneous coefficients p^j q^(n-j)) and writes the
//                         child operands in the interleaved level layout.
//   k_interp_top_rows<B>  CTA = 32 products x NP warps.  The child products y_k
//                         are staged through smem in chunks; warp j streams the
//                         coefficient row w_j = (sum_k A_jk y_k)/D_j (the
//                         even-odd + Newton listing program composed per row,
//                         PAPER.md:162) into smem; then the warps recompose
//                         w = sum_j w_j 2^(32 b j) segment by segment with a
//                         carry resolution between segments and write the
//                         row-major result.
#pragma once

namespace tg {

template <int B>
__host__ __device__ constexpr long long tg_evalc_cx(int k, int j) {
    return B == 3 ? tg_evalc_cx_T3(k, j) : tg_evalc_cx_T4(k, j);
}

template <int B>
__device__ __forceinline__ uint32_t rowstep(int j, const uint32_t (&y)[2 * B - 1], tg_rowstate& st) {
    if constexpr (B == 3) return tg_rowstep_T3(j, y, st);
    else return tg_rowstep_T4(j, y, st);
}

constexpr int TOP_CH = 16;   // limbs per staged chunk
#ifndef TG_ITS_CK
#define TG_ITS_CK 10   // k_interp_top_smem phase 1 chunk (C2, per-row code: 10 -> 207 us; 4: 241, 6: 230, 8: 230, 12: 275)
#endif

template <int B>
__global__ void __launch_bounds__(32 * (2 * B - 1)) k_eval_top_rows(
    const uint32_t* __restrict__ u, const uint32_t* __restrict__ v, uint32_t* __restrict__ U1,
    uint32_t* __restrict__ V1, size_t count, int n, int b, int e) {
    constexpr int NP = 2 * B - 1, G = 32, CH = (B == 8 ? 8 : TOP_CH), PP = 33;
    // (B = 8: the paper's points 0, +-2^i; values up to 2^42 u_j need 128-bit sums)
    using Acc = typename std::conditional<B == 8, __int128, long long>::type;
    // double-buffered chunks of CH limbs of every block of the G products,
    // filled with cp.async (zero-filled past a block's end) while the
    // previous chunk is evaluated
    __shared__ uint32_t S[2][2][B][CH][PP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t c0 = (size_t)blockIdx.x * G;
    const int nin = (int)min((size_t)G, count - c0);
    const size_t c = c0 + lane;
    const int lentop = n - (B - 1) * b;
    long long cf[B];
    if constexpr (B == 8) {
        // point 0 -> u_0; point 2i+1 -> +2^i; point 2i+2 -> -2^i (pointset_paper)
        const int i = (warp - 1) >> 1;
        const bool neg = warp > 0 && !(warp & 1);
#pragma unroll
        for (int j = 0; j < B; ++j)
            cf[j] = warp == 0 ? (j == 0 ? 1ll : 0ll) : ((neg && (j & 1)) ? -(1ll << (i * j)) : (1ll << (i * j)));
    } else {
#pragma unroll
        for (int j = 0; j < B; ++j) cf[j] = evalc<B>(warp, j);
    }
    const size_t stride_limb = (size_t)NP * count;
    auto stage = [&](int buf, int t0) {
        for (int idx = threadIdx.x; idx < 2 * G * B * CH; idx += blockDim.x) {
            const int tt = idx % CH;
            const int j = (idx / CH) % B;
            const int i = (idx / (CH * B)) % G;
            const int op = idx / (CH * B * G);
            const int t = t0 + tt;
            const int len = (j == B - 1) ? lentop : b;
            const bool ok = i < nin && t < len;
            const uint32_t* src = ok ? (op ? v : u) + (c0 + i) * (size_t)n + (size_t)j * b + t : u;
            const unsigned d = (unsigned)__cvta_generic_to_shared(&S[buf][op][j][tt][i]);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 4 : 0));
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    Acc au = 0, av = 0;
    const int nch = (e + CH - 1) / CH;
    stage(0, 0);
    for (int ci = 0; ci < nch; ++ci) {
        const int t0 = ci * CH;
        if (ci + 1 < nch) {
            stage((ci + 1) & 1, t0 + CH);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        if (lane < nin) {
            const int buf = ci & 1;
#pragma unroll 4
            for (int tt = 0; tt < CH; ++tt) {
                if (t0 + tt >= e) break;
                Acc lu = 0, lv = 0;
#pragma unroll
                for (int j = 0; j < B; ++j) {
                    lu += (Acc)cf[j] * (Acc)S[buf][0][j][tt][lane];
                    lv += (Acc)cf[j] * (Acc)S[buf][1][j][tt][lane];
                }
                lu += au;
                lv += av;
                const size_t o = (size_t)(t0 + tt) * stride_limb + (size_t)warp * count + c;
                U1[o] = (uint32_t)lu;
                V1[o] = (uint32_t)lv;
                au = lu >> 32;
                av = lv >> 32;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------------
// k_eval_top_p8: the top-level evaluation at the paper's Toom-8 points
// 0, +-2^i (i < 7; §4) of a batch (C3).  U(+-2^i) =
// E_i +- O_i with E_i = sum_{j even} u_j 2^(i j), O_i = sum_{j odd}
// u_j 2^(i j) (Eqs. 4.3-4.4): one thread per (product, operand, i) forms both
// points of the pair, limb t of each shifted block as one funnel shift of its
// limbs t - q and t - q - 1 (i j = 32 q + r), so there is no multiply; one
// thread per (product, operand) copies block 0 (point 0).  A half-warp holds
// the 16 tasks of one product (their loads of the same limbs coalesce into
// one request); outputs interleaved [e][15 count].
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(128) k_eval_top_p8(const uint32_t* __restrict__ u, const uint32_t* __restrict__ v,
                                                     uint32_t* __restrict__ U1, uint32_t* __restrict__ V1,
                                                     size_t count, int n, int b, int e) {
    constexpr int B = 8, NP = 15;
    const int task = threadIdx.x & 15;   // 0..6 pair i of u, 7..13 pair i of v, 14 / 15 point 0 of u / v
    const size_t c = (size_t)blockIdx.x * 8 + (threadIdx.x >> 4);
    if (c >= count) return;
    const bool opv = task == 15 || (task >= 7 && task < 14);
    const uint32_t* src = (opv ? v : u) + c * (size_t)n;
    uint32_t* out = (opv ? V1 : U1) + c;
    const size_t st = (size_t)NP * count;
    const int lentop = n - (B - 1) * b;
    if (task >= 14) {   // point 0: block 0
        for (int t = 0; t < e; ++t) out[(size_t)t * st] = t < b ? __ldg(src + t) : 0u;
        return;
    }
    const int i = opv ? task - 7 : task;
    uint32_t* op = out + (size_t)(2 * i + 1) * count;   // +2^i
    uint32_t* om = op + count;                          // -2^i
    int q[B], r[B];
    uint32_t h1[B], h2[B];
#pragma unroll
    for (int j = 0; j < B; ++j) {
        q[j] = (i * j) >> 5;
        r[j] = (i * j) & 31;
        h1[j] = h2[j] = 0u;
    }
    long long cp = 0, cm = 0;
    const bool v4 = ((b | n) & 3) == 0 && (((uintptr_t)src) & 15) == 0;
    // four limbs per step (one 16-byte load per block when aligned)
#pragma unroll 1
    for (int t0 = 0; t0 < e; t0 += 4) {
        uint32_t x[B][4];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            const int len = j == B - 1 ? lentop : b;
            const uint32_t* sp = src + (size_t)j * b + t0;
            if (v4 && t0 + 3 < len) {
                const uint4 w = __ldg(reinterpret_cast<const uint4*>(sp));
                x[j][0] = w.x; x[j][1] = w.y; x[j][2] = w.z; x[j][3] = w.w;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) x[j][k] = t0 + k < len ? __ldg(sp + k) : 0u;
            }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            if (t0 + k >= e) break;
            unsigned long long E = 0, O = 0;
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const uint32_t cur = q[j] ? h1[j] : x[j][k], prv = q[j] ? h2[j] : h1[j];
                const uint32_t sh = __funnelshift_l(prv, cur, r[j]);   // limb t of block j << (i j)
                h2[j] = h1[j];
                h1[j] = x[j][k];
                if (j & 1) O += sh;
                else E += sh;
            }
            const long long P = (long long)(E + O) + cp;
            const long long M = (long long)E - (long long)O + cm;
            const size_t o = (size_t)(t0 + k) * st;
            op[o] = (uint32_t)P;
            om[o] = (uint32_t)M;
            cp = P >> 32;
            cm = M >> 32;
        }
    }
}

// ------------------------------------------------------------------------
// k_eval_top_v4<B>: the top-level evaluation of k_eval_top_rows (B = 3, 4) with
// 16-byte staging and compile-time points.  CTA = 32 products x NP warps.
// Chunks of 16 limbs of every block of the 32 products are copied with 16-byte
// cp.async (zero-filled past a block's end) into S[op][j][i][16], the four
// 16-byte slots of row i XOR-swizzled by (i >> 1) & 3 so that the per-lane
// 16-byte reads of one slot are conflict-free; warp k streams U(x_k), V(x_k)
// with its homogeneous coefficients p^j q^(n-j) as immediates (one
// mad.wide.u32 per nonzero term); positions past every block (t >= b) carry
// only the running carry.  Requires n, b multiples of 4.
// ------------------------------------------------------------------------
template <int B, int K, bool SQ = false>
__device__ __forceinline__ void eval_top_v4_chunk(const uint32_t* __restrict__ Su, const uint32_t* __restrict__ Sv,
                                                  int lane, int t0, int tend, uint64_t& au, uint64_t& av,
                                                  uint32_t*& pu, uint32_t*& pv, size_t stride_limb) {
    constexpr int CH = 16;
    const int sw = (lane >> 1) & 3;
    // (rolled: seven point variants of one unrolled chunk overflow the
    // instruction cache)
#pragma unroll 1
    for (int q = 0; q < CH / 4; ++q) {
        if (t0 + 4 * q >= tend) break;
        uint4 xu[B], xv[B];
#pragma unroll
        for (int j = 0; j < B; ++j) {
            if (tg_evalc_cx<B>(K, j) != 0) {
                const int off = (j * 32 + lane) * CH + 4 * (q ^ sw);
                xu[j] = *reinterpret_cast<const uint4*>(Su + off);
                if constexpr (!SQ) xv[j] = *reinterpret_cast<const uint4*>(Sv + off);
            }
        }
#pragma unroll
        for (int r = 0; r < 4; ++r) {
            if (t0 + 4 * q + r >= tend) break;
            uint64_t lu = au, lv = av;
#pragma unroll
            for (int j = 0; j < B; ++j) {
                const long long cf = tg_evalc_cx<B>(K, j);
                if (cf == 0) continue;
                const uint32_t x = r == 0 ? xu[j].x : r == 1 ? xu[j].y : r == 2 ? xu[j].z : xu[j].w;
                if (cf > 0) lu = tg_madw((uint32_t)cf, x, lu);
                else lu = tg_msubw((uint32_t)(-cf), x, lu);
                if constexpr (!SQ) {
                    const uint32_t y = r == 0 ? xv[j].x : r == 1 ? xv[j].y : r == 2 ? xv[j].z : xv[j].w;
                    if (cf > 0) lv = tg_madw((uint32_t)cf, y, lv);
                    else lv = tg_msubw((uint32_t)(-cf), y, lv);
                }
            }
            *pu = (uint32_t)lu;
            pu += stride_limb;
            au = (uint64_t)((int64_t)lu >> 32);
            if constexpr (!SQ) {
                *pv = (uint32_t)lv;
                pv += stride_limb;
                av = (uint64_t)((int64_t)lv >> 32);
            }
        }
    }
}

#ifndef TG_EVAL_V4_MINB
#define TG_EVAL_V4_MINB 4   // 72 registers, four CTAs per SM (1: 122 registers, 91 us on C2; 4: 75 us)
#endif
// SQ: squaring (V = U): only u is staged and evaluated, V1 is not written
template <int B, bool SQ = false>
__global__ void __launch_bounds__(32 * (2 * B - 1), TG_EVAL_V4_MINB) k_eval_top_v4(
    const uint32_t* __restrict__ u, const uint32_t* __restrict__ v, uint32_t* __restrict__ U1,
    uint32_t* __restrict__ V1, size_t count, int n, int b, int e) {
    constexpr int NP = 2 * B - 1, G = 32, CH = 16, NQ = CH / 4;
    __shared__ __align__(16) uint32_t S[2][2][B][G][CH];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t c0 = (size_t)blockIdx.x * G;
    const int nin = (int)min((size_t)G, count - c0);
    const int lentop = n - (B - 1) * b;
    auto stage = [&](int buf, int t0) {
        constexpr int NE = (SQ ? 1 : 2) * B * G * NQ;
        for (int idx = threadIdx.x; idx < NE; idx += blockDim.x) {
            const int q = idx % NQ, i = (idx / NQ) % G, j = (idx / (NQ * G)) % B, op = idx / (NQ * G * B);
            const int t = t0 + 4 * q;
            const int len = (j == B - 1) ? lentop : b;
            const int words = (i < nin) ? min(max(len - t, 0), 4) : 0;
            const uint32_t* src = words ? (op ? v : u) + (c0 + i) * (size_t)n + (size_t)j * b + t : u;
            const unsigned d = (unsigned)__cvta_generic_to_shared(&S[buf][op][j][i][4 * (q ^ ((i >> 1) & 3))]);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(words * 4));
        }
        asm volatile("cp.async.commit_group;\n" ::: "memory");
    };
    const size_t stride_limb = (size_t)NP * count;
    uint32_t* pu = U1 + (size_t)warp * count + c0 + lane;
    uint32_t* pv = SQ ? nullptr : V1 + (size_t)warp * count + c0 + lane;
    uint64_t au = 0, av = 0;
    const int tb = min(b, e);                 // staged positions; [tb, e) are carries only
    const int nch = (tb + CH - 1) / CH;
    stage(0, 0);
    for (int ci = 0; ci < nch; ++ci) {
        const int t0 = ci * CH;
        if (ci + 1 < nch) {
            stage((ci + 1) & 1, t0 + CH);
            asm volatile("cp.async.wait_group 1;\n" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::: "memory");
        }
        __syncthreads();
        if (lane < nin) {
            const uint32_t* Su = &S[ci & 1][0][0][0][0];
            const uint32_t* Sv = &S[ci & 1][1][0][0][0];
            const int tend = min(t0 + CH, tb);
            switch (warp) {
                case 0: eval_top_v4_chunk<B, 0, SQ>(Su, Sv, lane, t0, tend, au, av, pu, pv, stride_limb); break;
                case 1: eval_top_v4_chunk<B, 1, SQ>(Su, Sv, lane, t0, tend, au, av, pu, pv, stride_limb); break;
                case 2: eval_top_v4_chunk<B, 2, SQ>(Su, Sv, lane, t0, tend, au, av, pu, pv, stride_limb); break;
                case 3: eval_top_v4_chunk<B, 3, SQ>(Su, Sv, lane, t0, tend, au, av, pu, pv, stride_limb); break;
                case 4: eval_top_v4_chunk<B, 4, SQ>(Su, Sv, lane, t0, tend, au, av, pu, pv, stride_limb); break;
                case 5: if constexpr (B >= 4) eval_top_v4_chunk<B, 5, SQ>(Su, Sv, lane, t0, tend, au, av, pu, pv, stride_limb); break;
                default: if constexpr (B >= 4) eval_top_v4_chunk<B, 6, SQ>(Su, Sv, lane, t0, tend, au, av, pu, pv, stride_limb); break;
            }
        }
        __syncthreads();
    }
    if (lane < nin) {
        for (int t = tb; t < e; ++t) {
            *pu = (uint32_t)au;
            pu += stride_limb;
            au = (uint64_t)((int64_t)au >> 32);
            if constexpr (!SQ) {
                *pv = (uint32_t)av;
                pv += stride_limb;
                av = (uint64_t)((int64_t)av >> 32);
            }
        }
    }
}

constexpr int ITOP_CH = 12;  // limb steps per staged chunk of the child products

__host__ __device__ inline size_t interp_top_rows_smem(int B, int Lw, int nseg) {
    const int NP = 2 * B - 1;
    return (size_t)4 * 32 * ((size_t)(NP - 2) * Lw + 2 * (size_t)NP * ITOP_CH + 4 * (size_t)nseg);
}

template <int B>
__global__ void __launch_bounds__(32 * (2 * B - 1)) k_interp_top_rows(
    const uint32_t* __restrict__ P1, uint32_t* __restrict__ w, size_t count, int ywidth, int Lw, int b, int wout,
    int nseg) {
    constexpr int NP = 2 * B - 1, G = 32, CH = ITOP_CH;
    extern __shared__ uint32_t sm[];
    uint32_t* W = sm;                              // rows 1..NP-2: [NP-2][Lw][32]
    uint32_t* Ys = W + (NP - 2) * Lw * G;          // 2 buffers x [NP][CH][32]
    uint32_t* CO = Ys + 2 * NP * CH * G;           // [nseg][32]
    uint32_t* L0 = CO + nseg * G;
    uint32_t* ON = L0 + nseg * G;
    uint32_t* CI = ON + nseg * G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t c0 = (size_t)blockIdx.x * G;
    const int nin = (int)min((size_t)G, count - c0);
    const size_t c = c0 + lane;
    const bool valid = lane < nin;
    const size_t S = (size_t)NP * count;           // limb stride of the child products

    // stage limbs [t0, t0+CH) of y_k for k in [k0, k1) into buffer `buf`
    auto stage = [&](int t0, int k0, int k1, int buf) {
        uint32_t* dst = Ys + buf * NP * CH * G;
        for (int k = k0; k < k1; ++k) {
            uint32_t fill = 0;
            if (valid) fill = (__ldg(P1 + (size_t)(ywidth - 1) * S + (size_t)k * count + c) >> 31) ? 0xFFFFFFFFu : 0u;
            uint32_t x[CH];
#pragma unroll
            for (int tt = 0; tt < CH; ++tt) {
                const int t = t0 + tt;
                x[tt] = 0;
                if (valid) x[tt] = (t < ywidth) ? __ldg(P1 + (size_t)t * S + (size_t)k * count + c) : fill;
            }
#pragma unroll
            for (int tt = 0; tt < CH; ++tt) dst[(k * CH + tt) * G + lane] = x[tt];
        }
    };
    // ---- phase 1: coefficient rows 1..NP-2 (rows 0 and NP-1 are y_0, y_inf).
    // Warps 0 and NP-1 are the loaders (double-buffered chunks), warps
    // 1..NP-2 compute their row from the current chunk.
    stage(0, warp, warp + 1, 0);
    __syncthreads();
    tg_rowstate st{0, 0, 0};
    const int nchunks = (Lw + 1 + CH - 1) / CH;
    for (int ci = 0; ci < nchunks; ++ci) {
        const int t0 = ci * CH;
        if (warp == 0) {
            if (ci + 1 < nchunks) stage(t0 + CH, 0, (NP + 1) / 2, (ci + 1) & 1);
        } else if (warp == NP - 1) {
            if (ci + 1 < nchunks) stage(t0 + CH, (NP + 1) / 2, NP, (ci + 1) & 1);
        } else if (valid) {
            const uint32_t* src = Ys + (ci & 1) * NP * CH * G;
            const int tmax = min(CH, Lw + 1 - t0);
            for (int tt = 0; tt < tmax; ++tt) {
                uint32_t y[NP];
#pragma unroll
                for (int k = 0; k < NP; ++k) y[k] = src[(k * CH + tt) * G + lane];
                const uint32_t r = rowstep<B>(warp, y, st);
                const int t = t0 + tt;
                if (t >= 1) W[((warp - 1) * Lw + t - 1) * G + lane] = r;
            }
        }
        __syncthreads();
    }

    // limb t of coefficient j (j = 0 and NP-1 straight from the products)
    auto wl = [&](int j, int t) -> uint32_t {
        if (j == 0 || j == NP - 1) return __ldg(P1 + (size_t)t * S + (size_t)j * count + c);
        return W[((j - 1) * Lw + t) * G + lane];
    };
    // segment s limb r (without carry): w_s[r] + w_{s-1}[b+r] + (r==0) w_{s-2}[2b];
    // every w_j >= 0 at the top level (sums of products of unsigned blocks)
    auto seg_sum = [&](int s, int r) -> uint64_t {
        uint64_t x = 0;
        if (s < NP) x += wl(s, r);
        if (s >= 1 && s - 1 < NP) x += wl(s - 1, b + r);
        if (r == 0 && s >= 2 && s - 2 < NP) x += wl(s - 2, 2 * b);
        return x;
    };
    constexpr int RU = 8;   // limbs per batch: loads issued before the carry chain
    // ---- phase 2: segment carry-outs
    if (valid) {
        for (int s = warp; s < nseg; s += NP) {
            const int len = min(b, wout - s * b);
            uint64_t carry = 0;
            uint32_t ones = 0xFFFFFFFFu, l0 = 0;
            for (int r0 = 0; r0 < len; r0 += RU) {
                uint64_t x[RU];
#pragma unroll
                for (int q = 0; q < RU; ++q) x[q] = (r0 + q < len) ? seg_sum(s, r0 + q) : 0;
#pragma unroll
                for (int q = 0; q < RU; ++q) {
                    if (r0 + q < len) {
                        const uint64_t y = carry + x[q];
                        const uint32_t lo = (uint32_t)y;
                        if (r0 + q == 0) l0 = lo; else ones &= lo;
                        carry = y >> 32;
                    }
                }
            }
            CO[s * G + lane] = (uint32_t)carry;
            L0[s * G + lane] = l0;
            ON[s * G + lane] = ones == 0xFFFFFFFFu;
        }
    }
    __syncthreads();
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
    // ---- phase 3: recompute each segment with its carry-in and write the row
    if (valid) {
        uint32_t* row = w + c * (size_t)wout;
        for (int s = warp; s < nseg; s += NP) {
            const int len = min(b, wout - s * b);
            uint64_t carry = CI[s * G + lane];
            for (int r0 = 0; r0 < len; r0 += RU) {
                uint64_t x[RU];
#pragma unroll
                for (int q = 0; q < RU; ++q) x[q] = (r0 + q < len) ? seg_sum(s, r0 + q) : 0;
#pragma unroll
                for (int q = 0; q < RU; ++q) {
                    if (r0 + q < len) {
                        const uint64_t y = carry + x[q];
                        row[s * b + r0 + q] = (uint32_t)y;
                        carry = y >> 32;
                    }
                }
            }
        }
    }
}

}  // namespace tg

namespace tg {

// ------------------------------------------------------------------------
// Top-level interpolation + recomposition in ONE streaming pass per product
// (steps a4 + a5; C1, C2).  The per-coefficient matrix form of the even-odd +
// listing program over the common denominator Dc = lcm D_j:
//     Dc * w = sum_j 2^(32 b j) N_j,   N_j = sum_k A'_jk y_k  (= Dc w_j >= 0)
// One thread per product streams w LSB-first: at output limb t = s b + r the
// rows j = s, s-1, s-2 contribute N_j limbs r, b + r, 2b + r, each row with
// its own signed carry chain (a chain ends after 2e limbs: N_j < 2^(32*2e));
// the three limb streams plus an unsigned carry give Dc*w, which is divided
// exactly by the odd part of Dc (2-adic inverse) and shifted by its power of
// two.  Products are read interleaved (coalesced across the warp); output
// limbs are staged per warp in shared memory and written row-major.
// ------------------------------------------------------------------------
template <int B> struct Comb;
template <> struct Comb<3> {
    static constexpr unsigned o = tg_combO_T3, inv = tg_combInv_T3;
    static constexpr int s = tg_combS_T3;
    __device__ static int A(int j, int k) { return (int)tg_combA_T3[j][k]; }
};
template <> struct Comb<4> {
    static constexpr unsigned o = tg_combO_T4, inv = tg_combInv_T4;
    static constexpr int s = tg_combS_T4;
    __device__ static int A(int j, int k) { return (int)tg_combA_T4[j][k]; }
};

constexpr int ITS_WARPS = 4;

template <int B>
__global__ void __launch_bounds__(32 * ITS_WARPS) k_interp_top_stream(const uint32_t* __restrict__ P1,
                                                                      uint32_t* __restrict__ w, size_t count,
                                                                      int ywidth, int b, int wout) {
    constexpr int NP = 2 * B - 1;
    __shared__ uint32_t stage[ITS_WARPS][32][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t c0w = (size_t)blockIdx.x * blockDim.x + (size_t)warp * 32;
    const size_t c = c0w + lane;
    const bool valid = c < count;
    const size_t S = (size_t)NP * count;
    const uint32_t* yb = P1 + (valid ? c : 0);
    const int X = ywidth - 2 * b;                 // limbs of y_k beyond 2b
    long long ca = 0, cb = 0, cc = 0;             // row carries (j = s, s-1, s-2)
    unsigned long long T = 0;                     // carry of the sum
    uint32_t bor = 0, qp = 0;
    uint32_t(*buf)[33] = stage[warp];
    const int nseg = wout / b + 1;                // covers limbs 0 .. wout (one extra for the shift)
    for (int s = 0; s <= nseg; ++s) {
        const bool hA = s < NP, hB = s >= 1 && s - 1 < NP, hC = s >= 2 && s - 2 < NP;
        int Aa[NP], Ab[NP], Ac[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) {
            Aa[k] = hA ? Comb<B>::A(s, k) : 0;
            Ab[k] = hB ? Comb<B>::A(s - 1, k) : 0;
            Ac[k] = hC ? Comb<B>::A(s - 2, k) : 0;
        }
        cc = cb;
        cb = ca;
        ca = 0;
        const int t0 = s * b;
        const int rmax = min(b, wout + 1 - t0);
        for (int r = 0; r < rmax; ++r) {
            long long la = ca, lb = cb, lc = cc;
            if (valid) {
#pragma unroll
                for (int k = 0; k < NP; ++k) {
                    const uint32_t* yk = yb + (size_t)k * count;
                    if (hA) la += (long long)Aa[k] * (long long)__ldg(yk + (size_t)r * S);
                    if (hB) lb += (long long)Ab[k] * (long long)__ldg(yk + (size_t)(b + r) * S);
                    if (hC && r < X) lc += (long long)Ac[k] * (long long)__ldg(yk + (size_t)(2 * b + r) * S);
                }
            }
            ca = la >> 32;
            cb = lb >> 32;
            unsigned long long x = T + (uint32_t)la + (uint32_t)lb;
            if (r < X) {
                cc = lc >> 32;
                x += (uint32_t)lc;
            }
            T = x >> 32;
            const uint32_t q = tg_divexact_step((uint32_t)x, bor, Comb<B>::inv, Comb<B>::o);
            const int t = t0 + r;
            if (t > 0) {
                const int e = t - 1;
                buf[e & 31][lane] = Comb<B>::s ? __funnelshift_r(qp, q, Comb<B>::s) : qp;
                if ((e & 31) == 31 || e == wout - 1) {
                    __syncwarp();
                    const int eb = e & ~31;
                    const int ncol = e - eb + 1;
                    for (int i = 0; i < 32; ++i) {
                        if (c0w + i < count && lane < ncol) w[(c0w + i) * (size_t)wout + eb + lane] = buf[lane][i];
                    }
                    __syncwarp();
                }
            }
            qp = q;
        }
    }
}

}  // namespace tg

namespace tg {

// ------------------------------------------------------------------------
// Top-level interpolation + recomposition with the products of a group of G
// instances resident in shared memory (steps a4 + a5; C1, C2):
//   phase 0  all threads: cp.async the 2B-1 products of the G instances,
//            [NP][2e][G] (each (limb, point) row is G contiguous words)
//   phase 1  warp j (1 <= j <= NP-2): stream the coefficient row
//            w_j = (sum_k A_jk y_k) / D_j (even-odd + listing program composed
//            per row) LSB-first, in lock-stepped chunks, and
//            write w_j in place over y_j (w_0 = y_0, w_2n = y_inf)
//   phase 2  recompose w = sum_j w_j 2^(32 b j) (Eq. 1.3) segment by segment:
//            local carries, one lane per instance resolves the carries between
//            segments, then the final limbs go to the row-major output.
// ------------------------------------------------------------------------
__host__ __device__ inline size_t interp_top_smem_bytes(int B, int ywidth, int G, int nseg) {
    return (size_t)4 * ((size_t)(2 * B - 1) * ywidth * G + 4 * (size_t)nseg * G);
}

// TMA bulk copies (cp.async.bulk, global -> shared) completing on an mbarrier
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* mb, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(count) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* mb, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* mb) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(mb))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* mb, unsigned phase) {
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n\t}\n" ::"r"(smem_u32(mb)),
        "r"(phase)
        : "memory");
}

__device__ __forceinline__ void cp_async4(uint32_t* dst_smem, const uint32_t* src) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst_smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(d), "l"(src));
}

// exactness check of row j (csrc/check.cuh): the products are read modulo
// 2^(32 ywidth), so a negative y_k adds -A_jk 2^(32 ywidth) to the dividend
template <int B>
__device__ __forceinline__ uint64_t row_sign_corr(int j, const uint32_t* Y, int ywidth, int G, int lane) {
    uint64_t corr = 0;
#pragma unroll
    for (int k = 0; k < 2 * B - 1; ++k)
        corr += (uint64_t)rowA<B>(j, k) * (Y[((size_t)k * ywidth + ywidth - 1) * G + lane] >> 31);
    return corr;
}

template <int B, int J>
__device__ __forceinline__ uint32_t rowstep_j(const uint32_t (&y)[2 * B - 1], tg_rowstate& st) {
    if constexpr (B == 3) {
        if constexpr (J == 1) return tg_rowstep_T3_1(y, st);
        else if constexpr (J == 2) return tg_rowstep_T3_2(y, st);
        else return tg_rowstep_T3_3(y, st);
    } else {
        if constexpr (J == 1) return tg_rowstep_T4_1(y, st);
        else if constexpr (J == 2) return tg_rowstep_T4_2(y, st);
        else if constexpr (J == 3) return tg_rowstep_T4_3(y, st);
        else if constexpr (J == 4) return tg_rowstep_T4_4(y, st);
        else return tg_rowstep_T4_5(y, st);
    }
}

// phase 1 of k_interp_top_smem for coefficient row J (every warp of the CTA
// runs the chunk loop so that the block barriers match; `work` = this warp
// owns row J).  Outputs of a chunk are written in place over y_J after all
// warps have read the chunk.
template <int B, int J>
__device__ __forceinline__ void interp_rows_inplace(uint32_t* Y, int ywidth, int G, int Lw, int lane, bool work) {
    constexpr int NP = 2 * B - 1, CK = TG_ITS_CK;
    const uint32_t* yb[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) yb[k] = Y + (size_t)k * ywidth * G + lane;
    uint32_t* dst = Y + (size_t)J * ywidth * G + lane;
    tg_rowstate st{0, 0, 0};
    for (int t0 = 0; t0 <= Lw; t0 += CK) {
        uint32_t ob[CK];
        if (work) {
#pragma unroll
            for (int tt = 0; tt < CK; ++tt) {
                const int t = t0 + tt;
                ob[tt] = 0;
                if (t <= Lw) {
                    const int off = t * G;
                    uint32_t y[NP];
#pragma unroll
                    for (int k = 0; k < NP; ++k) y[k] = yb[k][off];
                    ob[tt] = rowstep_j<B, J>(y, st);
                    if (t == 0) TG_CHECK_LOW(st.qp, rowS<B>(J));
                }
            }
        }
        __syncthreads();
        if (work) {
#pragma unroll
            for (int tt = 0; tt < CK; ++tt) {
                const int t = t0 + tt;
                if (t >= 1 && t <= Lw) dst[(t - 1) * G] = ob[tt];
            }
        }
        __syncthreads();
    }
    if (work && TG_CHECK_ENABLED) TG_CHECK_END(st.acc - row_sign_corr<B>(J, Y, ywidth, G, lane), st.bor, rowO<B>(J));
}

// YW_, G_, LW_, B_ != 0 fix ywidth, G, Lw and b at compile time (the C2 shape):
// every shared-memory offset of the unrolled chunk loops becomes an immediate.
template <int B, int YW_ = 0, int G_ = 0, int LW_ = 0, int B_ = 0>
__global__ void __launch_bounds__(32 * (2 * B - 1)) k_interp_top_smem(const uint32_t* __restrict__ P1,
                                                                       uint32_t* __restrict__ w, size_t count,
                                                                       int ywidth_, int Lw_, int b_, int wout, int G_arg,
                                                                       int nseg) {
    constexpr int NP = 2 * B - 1, CK = 16;
    const int ywidth = YW_ ? YW_ : ywidth_;
    const int Lw = LW_ ? LW_ : Lw_;
    const int b = B_ ? B_ : b_;
    const int G = G_ ? G_ : G_arg;
    extern __shared__ uint32_t sm[];
    uint32_t* Y = sm;                                   // [NP][ywidth][G]
    uint32_t* CO = Y + (size_t)NP * ywidth * G;         // [nseg][G]
    uint32_t* L0 = CO + nseg * G;
    uint32_t* ON = L0 + nseg * G;
    uint32_t* CI = ON + nseg * G;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t c0 = (size_t)blockIdx.x * G;
    const int nin = (int)min((size_t)G, count - c0);
    const size_t S = (size_t)NP * count;
    // ---- phase 0: rows (k, t) of G contiguous words; 16-byte cp.async when
    // aligned, several rows per warp instruction (one TMA bulk copy per
    // 112-byte row measured slower: 412 vs 392 us on C2)
    {
        const int nw = blockDim.x >> 5;
        const int nrows = NP * ywidth;
        const bool v16 = ((count & 3) == 0) && ((G & 3) == 0);
        if (v16) {
            const int q4 = G >> 2, rp = 32 / q4;
            const int sub = lane / q4, q = lane - sub * q4;
            if (sub < rp && nw == NP) {
                // rows in the source order R = t * NP + k: the stride NP * rp
                // keeps k fixed per thread and advances t by rp, so both
                // addresses are plain increments
                const int R0 = warp * rp + sub;
                const int k = R0 % NP;
                int t = R0 / NP;
                const int g = q * 4;
                const uint32_t* sr = P1 + (size_t)t * S + (size_t)k * count + c0 + g;
                uint32_t* dr = Y + (size_t)(k * ywidth + t) * G + g;
                const size_t sstep = (size_t)rp * S;
                const int dstep = rp * G;
                if (g + 3 < nin) {
                    unsigned d = (unsigned)__cvta_generic_to_shared(dr);
                    for (; t < ywidth; t += rp, sr += sstep, d += 4u * dstep)
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(sr));
                } else {
                    for (; t < ywidth; t += rp, sr += sstep, dr += dstep) {
#pragma unroll
                        for (int x = 0; x < 4; ++x) dr[x] = (g + x < nin) ? __ldg(sr + x) : 0u;
                    }
                }
            } else if (sub < rp) {
                // row R = k * ywidth + t, advanced incrementally (no division)
                const int stride = nw * rp;
                int R = warp * rp + sub;
                int k = R / ywidth, t = R - k * ywidth;
                for (; R < nrows; R += stride) {
                    const uint32_t* sr = P1 + (size_t)t * S + (size_t)k * count + c0;
                    uint32_t* dr = Y + (size_t)R * G;
                    const int g = q * 4;
                    if (g + 3 < nin) {
                        const unsigned d = (unsigned)__cvta_generic_to_shared(dr + g);
                        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(sr + g));
                    } else {
#pragma unroll
                        for (int x = 0; x < 4; ++x) dr[g + x] = (g + x < nin) ? __ldg(sr + g + x) : 0u;
                    }
                    t += stride;
                    while (t >= ywidth) { t -= ywidth; ++k; }
                }
            }
        } else {
            for (int R = warp; R < nrows; R += nw) {
                const int k = R / ywidth, t = R - k * ywidth;
                const uint32_t* sr = P1 + (size_t)t * S + (size_t)k * count + c0;
                uint32_t* dr = Y + (size_t)R * G;
                if (lane < G) {
                    if (lane < nin) cp_async4(dr + lane, sr + lane);
                    else dr[lane] = 0u;
                }
            }
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const bool act = lane < G;
    // warp 0 (idle in phase 1) writes recomposition segment 0 first: its limbs
    // are w_0[0..b) = y_0[0..b) alone, carry-out 0
    if (warp == 0 && act) {
        uint32_t* row0 = w + (c0 + lane) * (size_t)wout;
        const uint32_t* y0 = Y + lane;
        const int len = min(b, wout);
        if (lane < nin) {
            int r = 0;
            if ((wout & 3) == 0 && (((uintptr_t)w) & 15) == 0)
                for (; r + 4 <= len; r += 4)
                    *reinterpret_cast<uint4*>(row0 + r) =
                        make_uint4(y0[r * G], y0[(r + 1) * G], y0[(r + 2) * G], y0[(r + 3) * G]);
            for (; r < len; ++r) row0[r] = y0[r * G];
        }
        CO[lane] = 0u;
    }
    // ---- phase 1: rows 1..NP-2, in place (lock-stepped chunks; the barriers
    // are outside the per-lane work so every thread reaches them)
    // Toom-4: one specialised chunk loop per row (warp-uniform dispatch outside
    // the loop; idle warps run the barriers only).  C2: 277 -> 230 us.
#ifndef TG_ITS_NO_HOIST
    if constexpr (B == 4) {
        switch (warp) {
            case 1: interp_rows_inplace<B, 1>(Y, ywidth, G, Lw, lane, act); break;
            case 2: interp_rows_inplace<B, 2>(Y, ywidth, G, Lw, lane, act); break;
            case 3: interp_rows_inplace<B, 3>(Y, ywidth, G, Lw, lane, act); break;
            case 4: interp_rows_inplace<B, 4>(Y, ywidth, G, Lw, lane, act); break;
            case 5: interp_rows_inplace<B, 5>(Y, ywidth, G, Lw, lane, act); break;
            default: interp_rows_inplace<B, 1>(Y, ywidth, G, Lw, lane, false); break;
        }
    } else
#endif
    {
        constexpr int CK = TG_ITS_CK;   // limb positions per lock-stepped chunk
        const int j = warp;
        const bool rw = act && j >= 1 && j <= NP - 2;
        tg_rowstate st{0, 0, 0};
        for (int t0 = 0; t0 <= Lw; t0 += CK) {
            uint32_t ob[CK];
            if (rw) {
#pragma unroll
                for (int tt = 0; tt < CK; ++tt) {
                    const int t = t0 + tt;
                    ob[tt] = 0;
                    if (t <= Lw) {
                        uint32_t y[NP];
#pragma unroll
                        for (int k = 0; k < NP; ++k) y[k] = Y[(k * ywidth + t) * G + lane];
                        ob[tt] = rowstep<B>(j, y, st);
                        if (t == 0) TG_CHECK_LOW(st.qp, rowS<B>(j));
                    }
                }
            }
            __syncthreads();
            if (rw) {
#pragma unroll
                for (int tt = 0; tt < CK; ++tt) {
                    const int t = t0 + tt;
                    if (t >= 1 && t <= Lw) Y[(j * ywidth + t - 1) * G + lane] = ob[tt];
                }
            }
            __syncthreads();
        }
        if (rw && TG_CHECK_ENABLED) TG_CHECK_END(st.acc - row_sign_corr<B>(j, Y, ywidth, G, lane), st.bor, rowO<B>(j));
    }
    // ---- phase 2: recomposition (every w_j >= 0 at the top level).  Segment
    // s limb r = w_s[r] + w_{s-1}[b + r] (+ w_{s-2}[2b] at r = 0); absent rows
    // read a zero row of shared memory.
    __shared__ uint32_t zrow[32];
    if (threadIdx.x < 32) zrow[threadIdx.x] = 0u;
    __syncthreads();
    auto rowA = [&](int s) -> const uint32_t* { return s < NP ? Y + (size_t)(s * ywidth) * G + lane : nullptr; };
    auto rowB = [&](int s) -> const uint32_t* {
        return (s >= 1 && s - 1 < NP) ? Y + (size_t)((s - 1) * ywidth + b) * G + lane : nullptr;
    };
    auto extraC = [&](int s) -> uint32_t {
        return (s >= 2 && s - 2 < NP) ? Y[(size_t)((s - 2) * ywidth + 2 * b) * G + lane] : 0u;
    };
    // one pass: each segment is written with carry-in 0 (row-major, 16-byte
    // stores); the resolved carry-ins are added afterwards (they rarely ripple
    // past the segment's first limb)
    uint32_t* row = w + (c0 + lane) * (size_t)wout;
    const bool wr = act && lane < nin;
    if (act) {
        for (int s = warp + 1; s < nseg; s += NP) {   // segment 0 was written before phase 1
            const int len = min(b, wout - s * b);
            const uint32_t* pa = rowA(s);
            const uint32_t* pb = rowB(s);
            const int sa = pa ? G : 0, sb = pb ? G : 0;
            if (!pa) pa = zrow + lane;
            if (!pb) pb = zrow + lane;
            uint64_t carry = extraC(s);
            uint32_t ones = 0xFFFFFFFFu, l0 = 0;
            int r = 0;
            if (((s * b) & 3) == 0 && (wout & 3) == 0 && (((uintptr_t)w) & 15) == 0) {
                for (; r + 4 <= len; r += 4) {
                    uint32_t o[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const uint64_t y = carry + pa[(r + q) * sa] + pb[(r + q) * sb];
                        o[q] = (uint32_t)y;
                        carry = y >> 32;
                    }
                    if (r == 0) l0 = o[0]; else ones &= o[0];
                    ones &= o[1] & o[2] & o[3];
                    if (wr) *reinterpret_cast<uint4*>(row + s * b + r) = make_uint4(o[0], o[1], o[2], o[3]);
                }
            }
            for (; r < len; ++r) {
                const uint64_t y = carry + pa[r * sa] + pb[r * sb];
                const uint32_t lo = (uint32_t)y;
                if (r == 0) l0 = lo; else ones &= lo;
                if (wr) row[s * b + r] = lo;
                carry = y >> 32;
            }
            CO[s * G + lane] = (uint32_t)carry;
            L0[s * G + lane] = l0;
            ON[s * G + lane] = ones == 0xFFFFFFFFu;
        }
    }
    __syncthreads();
    if (act && warp == 0) {
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
    if (wr) {
        for (int s = warp + 1; s < nseg; s += NP) {
            uint32_t cin = CI[s * G + lane];
            const int len = min(b, wout - s * b);
            for (int r = 0; r < len && cin; ++r) {
                const uint32_t x = row[s * b + r];
                const uint32_t y = x + cin;
                row[s * b + r] = y;
                cin = (y < x) ? 1u : 0u;
            }
        }
    }
}

}  // namespace tg

namespace tg {

// ------------------------------------------------------------------------
// Top-level interpolation + recomposition, ONE WARP PER PRODUCT (steps a4 +
// a5; C1, C2).  The combined matrix form over the common denominator Dc
// (PAPER.md:162 + Eq. 1.3, reading 12):
//     Dc * w = sum_j 2^(32 b j) sum_k A'_jk y_k
// The warp stages the 2B-1 products y_k (row-major, coalesced) in shared
// memory; lane L forms positions [L*CH, L*CH+CH) of the linear combination,
// normalises them locally and the carry / 2-adic borrow of the exact division
// by the odd part of Dc is resolved with a warp scan of the composable
// carry/borrow maps (csrc/longvec.cuh); then the quotient is shifted by the
// power of two of Dc and stored coalesced.  y_k are sign-extended (their
// fills enter as per-row constants).
// ------------------------------------------------------------------------
struct WarpInterpConst {
    uint32_t o, oinv, p32, Mch, mi;
    unsigned long long orcp;
    int sh;
};

template <int B, int CH>
__global__ void __launch_bounds__(256) k_interp_top_warp(const uint32_t* __restrict__ P1, uint32_t* __restrict__ w,
                                                         size_t count, int ywidth, int b, int wout, WarpInterpConst K) {
    constexpr int NP = 2 * B - 1;
    extern __shared__ uint32_t wsm[];
    __shared__ long long sA[NP][NP];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x < NP * NP) {
        const int j = threadIdx.x / NP, k = threadIdx.x % NP;
        sA[j][k] = (B == 3) ? tg_combA_T3[j][k] : tg_combA_T4[j][k];
    }
    const size_t c = (size_t)blockIdx.x * nw + warp;
    const int P = wout + 1;                       // positions 0..wout (one extra for the shift)
    const int ysz = max(NP * ywidth, 64 * CH);     // products, later the 64-bit transpose scratch
    const int wstride = (ysz + 32 * CH + 1 + 3) & ~3;
    uint32_t* Ys = wsm + (size_t)warp * wstride;
    uint32_t* Qs = Ys + ysz;
    long long* Fs = reinterpret_cast<long long*>(wsm + (size_t)nw * wstride) + warp * NP;
    __syncthreads();
    if (c >= count) return;                       // warp-uniform
    // stage the products (row k*count + c of the row-major [NP*count][ywidth] buffer)
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const uint32_t* src = P1 + ((size_t)k * count + c) * ywidth;
        for (int i = lane; i < ywidth; i += 32) Ys[k * ywidth + i] = __ldg(src + i);
    }
    __syncwarp();
    long long fillv[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) fillv[k] = (Ys[k * ywidth + ywidth - 1] >> 31) ? 0xFFFFFFFFll : 0ll;
    const int p0 = lane * CH;
    long long lin[CH];
    {
        // pass 1: positions p = lane + 32 q (the warp covers 32 consecutive
        // positions per q, so the set of active rows j is warp-uniform);
        // rows entirely past their products add the constant F_j.
        if (lane < NP) {
            long long f = 0;
#pragma unroll
            for (int k = 0; k < NP; ++k) f += sA[lane][k] * fillv[k];
            Fs[lane] = f;
        }
        __syncwarp();
        const long long* F = Fs;
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int pw = 32 * q;                  // first position of this row of the warp
            const int p = pw + lane;
            // rows with b*j <= p (started) and p - b*j < ywidth (not yet past)
            const int jhi = min(NP - 1, (pw + 31) / b);
            const int jlo = max(0, (pw - ywidth) / b);   // rows below jlo are past for the whole warp row
            long long acc = 0;
            for (int j = 0; j < jlo; ++j) acc += F[j];
            for (int j = jlo; j <= jhi; ++j) {
                const int i = p - b * j;
                if (i >= ywidth) {
                    acc += F[j];
                } else if (i >= 0) {
                    long long sj = 0;
#pragma unroll
                    for (int k = 0; k < NP; ++k) sj += sA[j][k] * (long long)Ys[k * ywidth + i];
                    acc += sj;
                }
            }
            lin[q] = acc;
        }
    }
    // transpose through shared memory: lane L takes positions [L*CH, L*CH+CH)
    {
        long long* T64 = reinterpret_cast<long long*>(Ys);   // the products are no longer needed
        __syncwarp();
#pragma unroll
        for (int q = 0; q < CH; ++q) T64[32 * q + lane] = lin[q];
        __syncwarp();
#pragma unroll
        for (int q = 0; q < CH; ++q) lin[q] = T64[p0 + q];
        __syncwarp();
    }
    // local normalisation -> this lane's carry / borrow map
    const LMod M{K.o, K.orcp};
    uint32_t x[CH];
    long long cy = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const long long v = lin[q] + cy;
        x[q] = (uint32_t)v;
        cy = v >> 32;
    }
    LAgg A;
    {
        const unsigned long long L64 = (unsigned long long)x[0] | ((unsigned long long)x[1] << 32);
        bool tz = true, to = true;
#pragma unroll
        for (int q = 2; q < CH; ++q) { tz &= (x[q] == 0u); to &= (x[q] == 0xFFFFFFFFu); }
        A.lo = (tz && L64 <= 0x8000000000000000ull) ? (long long)(0ull - L64) : LLONG_MIN;
        const unsigned long long comp = 0ull - L64;
        A.hi = (to && L64 != 0 && comp <= (unsigned long long)LLONG_MAX) ? (long long)comp : LLONG_MAX;
        A.cout[0] = cy - 1;
        A.cout[1] = cy;
        A.cout[2] = cy + 1;
        uint32_t r = 0;
#pragma unroll
        for (int q = CH - 1; q >= 0; --q) r = lv_mod((unsigned long long)r * K.p32 + x[q], M);
        A.m = K.mi;
#pragma unroll
        for (int p = 0; p < 3; ++p) {
            const unsigned long long t = (unsigned long long)(K.o - r) + (p == 2 ? K.Mch : 0u) + (p == 0 ? (K.o - K.Mch) : 0u);
            A.g[p] = lv_mulmod(lv_mod(t, M), K.mi, M);
        }
    }
    LAgg inc = A;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const LAgg prev = lv_shfl_up(inc, d);
        if (lane >= d) inc = lv_compose(prev, inc, M);
    }
    const LAgg excl = lv_shfl_up(inc, 1);
    long long cin = 0;
    uint32_t bin = 0;
    if (lane > 0) lv_apply(excl, cin, bin, M);
    // exact limbs, exact division by the odd part of Dc
    cy = cin;
    uint32_t beta = bin;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const long long v = lin[q] + cy;
        cy = v >> 32;
        Qs[p0 + q] = tg_divexact_step((uint32_t)v, beta, K.oinv, K.o);
    }
    __syncwarp();
    // shift by the power of two of Dc, coalesced row-major store
    uint32_t* row = w + c * (size_t)wout;
    for (int t = lane; t < wout; t += 32) {
        const uint32_t lo = Qs[t];
        row[t] = K.sh ? __funnelshift_r(lo, Qs[t + 1], K.sh) : lo;
    }
    (void)P;
}

inline size_t interp_top_warp_smem(int B, int ywidth, int CH, int wpb) {
    const int ysz = std::max((2 * B - 1) * ywidth, 64 * CH);
    const int wstride = (ysz + 32 * CH + 1 + 3) & ~3;
    return (size_t)4 * wpb * wstride + (size_t)8 * wpb * (2 * B - 1);
}

}  // namespace tg

namespace tg {

// ------------------------------------------------------------------------
// Top-level interpolation of the paper's Toom-8 (C3) with one thread per
// (coefficient row, product) instead of per product: the per-coefficient
// rows w_j = (sum_k m_jk y_k) / (2^s_j o1_j o2_j) composed from the even-odd
// + listing program (generator emit_bigrow_tables), streamed
// LSB-first with a 64-bit carry, two 2-adic exact divisions by the odd word
// factors and the exact right shift.  Rows go to the scratch W [NP][Lw][count]
// (row 0 = y_0 is not copied); then the recomposition w = sum_j w_j 2^(32bj)
// (Eq. 1.3) runs one thread per (segment, product) with carry-in 0, and one
// thread per product resolves the segment carries and adds them.
// ------------------------------------------------------------------------
__global__ void __launch_bounds__(128, 4) k_interp_rows_p8(const uint32_t* __restrict__ P1, uint32_t* __restrict__ W,
                                                         size_t count, int ywidth, int Lw) {
    constexpr int NP = 15;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)(NP - 1) * count) return;
    const int j = 1 + (int)(idx / count);
    const size_t c = idx - (size_t)(j - 1) * count;
    const size_t S = (size_t)NP * count;
    const uint32_t* yb = P1 + c;
    long long m[NP];
    uint32_t fill[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        m[k] = tg_brow_m_P8[j][k];
        fill[k] = (__ldg(yb + (size_t)(ywidth - 1) * S + (size_t)k * count) >> 31) ? 0xFFFFFFFFu : 0u;
    }
    // exactness check: the window holds y_k mod 2^(32 window), a negative y_k
    // adds -m_k 2^(32 window) to the dividend (csrc/check.cuh)
    long long corr = 0;
    if (tg_check_on) {
#pragma unroll
        for (int k = 0; k < NP; ++k) corr += m[k] * (long long)(fill[k] & 1u);
    }
    const uint32_t o1 = tg_brow_o1_P8[j], o2 = tg_brow_o2_P8[j], i1 = tg_brow_i1_P8[j], i2 = tg_brow_i2_P8[j];
    const int sh = tg_brow_s_P8[j], a = sh >> 5, r = sh & 31;
    long long acc = 0;
    uint32_t b1 = 0, b2 = 0, qp = 0;
    uint32_t* dst = W + (size_t)j * Lw * count + c;
    const int tend = Lw + a + (r ? 1 : 0);
    // limbs of the 15 products, two limbs ahead in registers
    auto ld = [&](int t, uint32_t (&y)[NP]) {
        if (t < ywidth) {
            const uint32_t* yt = yb + (size_t)t * S;
#pragma unroll
            for (int k = 0; k < NP; ++k) y[k] = __ldg(yt + (size_t)k * count);
        } else {
#pragma unroll
            for (int k = 0; k < NP; ++k) y[k] = fill[k];
        }
    };
    uint32_t y0[NP], y1[NP];
    ld(0, y0);
    ld(1, y1);
    // with the exactness check on, the chains run 3 limbs further so that the
    // whole dividend (up to o1 o2 < 2^64 times the quotient) is inside the window
    const int tlast = tend + (tg_check_on ? 3 : 0);
#pragma unroll 1
    for (int t = 0; t < tlast; ++t) {
        uint32_t y[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) { y[k] = y0[k]; y0[k] = y1[k]; }
        ld(t + 2, y1);
        __int128 lin = acc;
#pragma unroll
        for (int k = 0; k < NP; ++k) lin += (__int128)m[k] * (__int128)y[k];
        acc = (long long)(lin >> 32);
        uint32_t q = tg_divexact_step((uint32_t)lin, b1, i1, o1);
        if (o2 > 1) q = tg_divexact_step(q, b2, i2, o2);
        // quotient limb t; output limb u = t - a (r = 0) or t - a - 1 (r > 0)
        const int u = t - a - (r ? 1 : 0);
        if (u >= 0 && u < Lw) dst[(size_t)u * count] = r ? __funnelshift_r(qp, q, r) : q;
        if (t <= a && tg_check_on) tg_check_low(t < a ? (q ? 1u : 0u) : q, t < a ? 1 : r);   // exact 2^sh
        qp = q;
    }
    if (tg_check_on) {
        // the dividend ended (tend >= its length): carry 0 / -1, borrows 0 / o-1
        // the tlast-limb window holds y_k mod 2^(32 tlast): negative y_k add
        // -m_k 2^(32 tlast) (csrc/check.cuh); the first quotient's own carry
        // past the window is then (acc - b1) / o1
        const long long ac = acc - corr;
        tg_check_end((uint64_t)ac, b1, o1);
        if (o2 > 1) tg_check_end((uint64_t)((ac - (long long)b1) / (long long)o1), b2, o2);
    }
}

// The same rows with the multipliers as compile-time constants: |m_jk| =
// h 2^27 + l, each part one IMAD.WIDE.U32 (immediate x limb) into 64-bit sums
// separated by the sign of m_jk (every sum < 2^61: toomgen asserts it), so a
// row limb costs 2 multiply-adds per term instead of a generic 64 x 32 -> 128
// multiply.  The linear combination, carries, divisions and output are those
// of k_interp_rows_p8 (the same integers).  One CTA = one row x 128
// products (CTA-uniform row constants).
template <int J, int K>
__device__ __forceinline__ void p8s_term(uint32_t y, uint64_t& lp, uint64_t& hp, uint64_t& ln, uint64_t& hn) {
    constexpr long long M = tg_brow_cx_P8(J, K);
    constexpr unsigned long long A = M < 0 ? (unsigned long long)(-M) : (unsigned long long)M;
    constexpr uint32_t L = (uint32_t)(A & ((1ull << tg_brow_split_P8) - 1)), H = (uint32_t)(A >> tg_brow_split_P8);
    static_assert((A >> tg_brow_split_P8) < (1ull << 32), "27-bit split: high part one word");
    if constexpr (M > 0) {
        if constexpr (L != 0) lp = tg_madw(L, y, lp);
        if constexpr (H != 0) hp = tg_madw(H, y, hp);
    } else if constexpr (M < 0) {
        if constexpr (L != 0) ln = tg_madw(L, y, ln);
        if constexpr (H != 0) hn = tg_madw(H, y, hn);
    }
}
template <int J, int K = 0>
__device__ __forceinline__ void p8s_terms(const uint32_t (&y)[15], uint64_t& lp, uint64_t& hp, uint64_t& ln, uint64_t& hn) {
    if constexpr (K < 15) {
        p8s_term<J, K>(y[K], lp, hp, ln, hn);
        p8s_terms<J, K + 1>(y, lp, hp, ln, hn);
    }
}
template <int J>
__device__ __forceinline__ void p8s_row(const uint32_t* __restrict__ P1, uint32_t* __restrict__ W, size_t count, size_t c,
                                        int ywidth, int Lw) {
    constexpr int NP = 15;
    const size_t S = (size_t)NP * count;
    const uint32_t* yb = P1 + c;
    uint32_t fill[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) fill[k] = (__ldg(yb + (size_t)(ywidth - 1) * S + (size_t)k * count) >> 31) ? 0xFFFFFFFFu : 0u;
    long long corr = 0;   // exactness check: a negative y_k read modulo 2^(32 window) adds -m_k 2^(32 window)
    if (tg_check_on) {
#pragma unroll
        for (int k = 0; k < NP; ++k) corr += tg_brow_cx_P8(J, k) * (long long)(fill[k] & 1u);
    }
    const uint32_t o1 = tg_brow_o1_P8[J], o2 = tg_brow_o2_P8[J], i1 = tg_brow_i1_P8[J], i2 = tg_brow_i2_P8[J];
    const int sh = tg_brow_s_P8[J], a = sh >> 5, r = sh & 31;
    long long acc = 0;
    uint32_t b1 = 0, b2 = 0, qp = 0;
    uint32_t* dst = W + (size_t)J * Lw * count + c;
    const int tend = Lw + a + (r ? 1 : 0);
    auto ld = [&](int t, uint32_t (&y)[NP]) {
        if (t < ywidth) {
            const uint32_t* yt = yb + (size_t)t * S;
#pragma unroll
            for (int k = 0; k < NP; ++k) y[k] = __ldg(yt + (size_t)k * count);
        } else {
#pragma unroll
            for (int k = 0; k < NP; ++k) y[k] = fill[k];
        }
    };
    const int tlast = tend + (tg_check_on ? 3 : 0);
    auto step = [&](int t, const uint32_t (&y)[NP]) {
        uint64_t lp = 0, hp = 0, ln = 0, hn = 0;
        p8s_terms<J>(y, lp, hp, ln, hn);
        const __int128 lin = (__int128)(long long)(lp - ln) + ((__int128)(long long)(hp - hn) << tg_brow_split_P8) + acc;
        acc = (long long)(lin >> 32);
        uint32_t q = tg_divexact_step((uint32_t)lin, b1, i1, o1);
        if (o2 > 1) q = tg_divexact_step(q, b2, i2, o2);
        const int u = t - a - (r ? 1 : 0);
        if (u >= 0 && u < Lw) {   // output limbs in order: one pointer step each
            *dst = r ? __funnelshift_r(qp, q, r) : q;
            dst += count;
        }
        if (t <= a && tg_check_on) tg_check_low(t < a ? (q ? 1u : 0u) : q, t < a ? 1 : r);
        qp = q;
    };
    // three limbs in flight: buffer X is refilled for limb t + 3 right after
    // limb t used it (no register moves between the load and its use)
    uint32_t yA[NP], yB[NP], yC[NP];
    ld(0, yA);
    ld(1, yB);
    ld(2, yC);
#pragma unroll 1
    for (int t = 0; t < tlast; t += 3) {
        step(t, yA);
        ld(t + 3, yA);
        if (t + 1 >= tlast) break;
        step(t + 1, yB);
        ld(t + 4, yB);
        if (t + 2 >= tlast) break;
        step(t + 2, yC);
        ld(t + 5, yC);
    }
    if (tg_check_on) {
        const long long ac = acc - corr;
        tg_check_end((uint64_t)ac, b1, o1);
        if (o2 > 1) tg_check_end((uint64_t)((ac - (long long)b1) / (long long)o1), b2, o2);
    }
}
__global__ void __launch_bounds__(128) k_interp_rows_p8s(const uint32_t* __restrict__ P1, uint32_t* __restrict__ W,
                                                         size_t count, int ywidth, int Lw) {
    const unsigned nb = (unsigned)((count + 127) / 128);   // CTAs per row
    const int row = 1 + (int)(blockIdx.x / nb);
    const size_t c = (size_t)(blockIdx.x % nb) * 128 + threadIdx.x;
    if (c >= count) return;
    switch (row) {
        case 1: p8s_row<1>(P1, W, count, c, ywidth, Lw); break;
        case 2: p8s_row<2>(P1, W, count, c, ywidth, Lw); break;
        case 3: p8s_row<3>(P1, W, count, c, ywidth, Lw); break;
        case 4: p8s_row<4>(P1, W, count, c, ywidth, Lw); break;
        case 5: p8s_row<5>(P1, W, count, c, ywidth, Lw); break;
        case 6: p8s_row<6>(P1, W, count, c, ywidth, Lw); break;
        case 7: p8s_row<7>(P1, W, count, c, ywidth, Lw); break;
        case 8: p8s_row<8>(P1, W, count, c, ywidth, Lw); break;
        case 9: p8s_row<9>(P1, W, count, c, ywidth, Lw); break;
        case 10: p8s_row<10>(P1, W, count, c, ywidth, Lw); break;
        case 11: p8s_row<11>(P1, W, count, c, ywidth, Lw); break;
        case 12: p8s_row<12>(P1, W, count, c, ywidth, Lw); break;
        case 13: p8s_row<13>(P1, W, count, c, ywidth, Lw); break;
        default: p8s_row<14>(P1, W, count, c, ywidth, Lw); break;
    }
}

// recomposition pass 1: thread per (segment s, product c), carry-in 0.
// Coefficient j: w_0 = y_0 and (last_copy) w_{NP-1} = y_inf come from the
// products (interleaved [ywidth][NP*count]), the others from W [NP][Lw][count];
// every w_j is an exact two's-complement value of Lw limbs (sign-extended past
// them: below the top level they can be negative).  Segment s limb r sums
// w_s[r] + w_{s-1}[b + r] + w_{s-2}[2b + r] (+ the fills of the rows that have
// ended); the output limb goes to out[c*out_is + t*out_ls]; R[3][nseg][count]
// receives the carry-out, limb 0 and whether limbs 1.. are all ones.
struct RecompArgs {
    const uint32_t* P1;
    const uint32_t* W;
    uint32_t* out;
    long long out_is, out_ls;
    uint32_t* R;
    size_t count;
    int NP, Lw, b, wout, nseg, last_copy;
};

__global__ void __launch_bounds__(128) k_recomp_seg(RecompArgs A) {
    const size_t count = A.count;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)A.nseg * count) return;
    const int s = (int)(idx / count);
    const size_t c = idx - (size_t)s * count;
    const int NP = A.NP, Lw = A.Lw, b = A.b;
    const size_t S = (size_t)NP * count;
    auto fromY = [&](int j) { return j == 0 || (A.last_copy && j == NP - 1); };
    auto wl = [&](int j, int t) -> uint32_t {
        return fromY(j) ? __ldg(A.P1 + (size_t)t * S + (size_t)j * count + c) : __ldg(A.W + ((size_t)j * Lw + t) * count + c);
    };
    auto fillj = [&](int j) -> uint32_t { return wl(j, Lw - 1) >> 31; };
    uint32_t lowfills = 0, fillC = 0;
    for (int j = 0; j <= s - 2 && j < NP; ++j) {
        const uint32_t f = fillj(j);
        if (j == s - 2) fillC = f;
        else lowfills += f;
    }
    const int len = min(b, A.wout - s * b);
    const bool hA = s < NP, hB = s >= 1 && s - 1 < NP, hC = s >= 2 && s - 2 < NP;
    // per-limb constants: limb 0 gets the ended rows' fills and w_{s-2}[2b];
    // limbs 1.. also the fill of w_{s-2} (its last limb is 2b)
    const uint64_t k0 = (uint64_t)lowfills * 0xFFFFFFFFull + (hC ? wl(s - 2, 2 * b) : 0u);
    const uint64_t k1 = (uint64_t)(lowfills + fillC) * 0xFFFFFFFFull;
    uint64_t carry = 0;
    uint32_t ones = 0xFFFFFFFFu, l0 = 0;
    uint32_t* o = A.out + (long long)c * A.out_is + (long long)s * b * A.out_ls;
    const bool v4 = A.out_ls == 1 && ((reinterpret_cast<uintptr_t>(o)) & 15) == 0;
    constexpr int RQ = 8;   // limbs loaded ahead (4: 121 us on C3, latency-bound at 21 % warps active)
    for (int r0 = 0; r0 < len; r0 += RQ) {
        uint32_t xa[RQ], xb[RQ];
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
            xa[q] = (hA && r0 + q < len) ? wl(s, r0 + q) : 0u;
            xb[q] = (hB && r0 + q < len) ? wl(s - 1, b + r0 + q) : 0u;
        }
        uint32_t z[RQ];
#pragma unroll
        for (int q = 0; q < RQ; ++q) {
            z[q] = 0u;
            if (r0 + q < len) {
                const uint64_t y = carry + xa[q] + xb[q] + (r0 + q > 0 ? k1 : k0);
                const uint32_t lo = (uint32_t)y;
                if (r0 + q == 0) l0 = lo; else ones &= lo;
                z[q] = lo;
                carry = y >> 32;
            }
        }
        if (v4 && r0 + RQ <= len) {   // row-major output: one 32-byte sector per thread and step
            uint4* o4 = reinterpret_cast<uint4*>(o + r0);
            o4[0] = make_uint4(z[0], z[1], z[2], z[3]);
            o4[1] = make_uint4(z[4], z[5], z[6], z[7]);
        } else {
#pragma unroll
            for (int q = 0; q < RQ; ++q)
                if (r0 + q < len) o[(long long)(r0 + q) * A.out_ls] = z[q];
        }
    }
    A.R[(size_t)s * count + c] = (uint32_t)carry;
    A.R[((size_t)A.nseg + s) * count + c] = l0;
    A.R[((size_t)2 * A.nseg + s) * count + c] = ones == 0xFFFFFFFFu;
}

// recomposition pass 2: thread per product: resolve the segment carries
// (the carry-in of segment s replaces its carry-out in R)
__global__ void __launch_bounds__(128) k_recomp_fix(uint32_t* __restrict__ R, size_t count, int nseg) {
    const size_t c = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= count) return;
    uint32_t cin = 0;
    for (int s0 = 0; s0 < nseg; s0 += 8) {   // the records of 8 segments loaded ahead of the chain
        uint32_t co[8], l0[8], on[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const bool in = s0 + q < nseg;
            co[q] = in ? R[(size_t)(s0 + q) * count + c] : 0u;
            l0[q] = in ? R[((size_t)nseg + s0 + q) * count + c] : 0u;
            on[q] = in ? R[((size_t)2 * nseg + s0 + q) * count + c] : 0u;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (s0 + q < nseg) {
                uint32_t cout = co[q];
                if (cin && l0[q] + cin < l0[q] && on[q]) cout += 1;
                R[(size_t)(s0 + q) * count + c] = cin;
                cin = cout;
            }
        }
    }
}

// recomposition pass 3: thread per (segment, product): add the carry-in (it
// ripples through all-ones limbs, e.g. the all-ones operands of C3)
__global__ void __launch_bounds__(128) k_recomp_apply(RecompArgs A) {
    const size_t count = A.count;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)A.nseg * count) return;
    const int s = (int)(idx / count);
    const size_t c = idx - (size_t)s * count;
    uint32_t cc = A.R[(size_t)s * count + c];
    if (!cc) return;
    uint32_t* o = A.out + (long long)c * A.out_is + (long long)s * A.b * A.out_ls;
    const int len = min(A.b, A.wout - s * A.b);
    {
        // the carry wraps limb 0 and every other limb is all ones (pass 1's
        // records; C3's all-ones quarter): the segment becomes limb 0 + carry
        // and zeros, stored without reading it back
        const uint32_t l0 = A.R[((size_t)A.nseg + s) * count + c];
        if (l0 + cc < l0 && A.R[((size_t)2 * A.nseg + s) * count + c]) {
            o[0] = l0 + cc;
            int r = 1;
            if (A.out_ls == 1 && ((reinterpret_cast<uintptr_t>(o)) & 15) == 0) {   // 16-byte zero stores
                for (; r < 4 && r < len; ++r) o[r] = 0u;
                for (; r + 4 <= len; r += 4) *reinterpret_cast<uint4*>(o + r) = make_uint4(0u, 0u, 0u, 0u);
            }
            for (; r < len; ++r) o[(long long)r * A.out_ls] = 0u;
            return;
        }
    }
    // 8 limbs loaded ahead of the ripple (one load -> store chain per limb
    // was a serial run of L2 latencies: 53 us on C3's all-ones quarter)
    for (int r = 0; r < len && cc; r += 8) {
        uint32_t x[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q] = (r + q < len) ? o[(long long)(r + q) * A.out_ls] : 0u;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            if (r + q < len && cc) {
                const uint32_t y = x[q] + cc;
                o[(long long)(r + q) * A.out_ls] = y;
                cc = (y < x[q]) ? 1u : 0u;
            }
        }
    }
}

// Toom-3/4 coefficient rows, one thread per (row j in 1..NP-2, product):
// w_j = (sum_k A_jk y_k) / (o_j 2^s_j) streamed LSB-first (the generated row
// steps), y_k from the interleaved products two limbs ahead in registers,
// w_j to W [NP][Lw][count].  With k_recomp_* this is the row-parallel
// interpolation + recomposition of a batched level.
template <int B>
__global__ void __launch_bounds__(128) k_interp_rows_w(const uint32_t* __restrict__ P1, uint32_t* __restrict__ W,
                                                        size_t count, int ywidth, int Lw) {
    constexpr int NP = 2 * B - 1;
    const size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (size_t)(NP - 2) * count) return;
    const int j = 1 + (int)(idx / count);
    const size_t c = idx - (size_t)(j - 1) * count;
    const size_t S = (size_t)NP * count;
    const uint32_t* yb = P1 + c;
    uint32_t fill[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) fill[k] = (__ldg(yb + (size_t)(ywidth - 1) * S + (size_t)k * count) >> 31) ? 0xFFFFFFFFu : 0u;
    auto ld = [&](int t, uint32_t (&y)[NP]) {
        if (t < ywidth) {
            const uint32_t* yt = yb + (size_t)t * S;
#pragma unroll
            for (int k = 0; k < NP; ++k) y[k] = __ldg(yt + (size_t)k * count);
        } else {
#pragma unroll
            for (int k = 0; k < NP; ++k) y[k] = fill[k];
        }
    };
    uint32_t* dst = W + (size_t)j * Lw * count + c;
    tg_rowstate st{0, 0, 0};
    uint32_t y0[NP], y1[NP];
    ld(0, y0);
    ld(1, y1);
#pragma unroll 1
    for (int t = 0; t <= Lw; ++t) {
        uint32_t y[NP];
#pragma unroll
        for (int k = 0; k < NP; ++k) { y[k] = y0[k]; y0[k] = y1[k]; }
        ld(t + 2, y1);
        const uint32_t r = rowstep<B>(j, y, st);
        if (t >= 1) dst[(size_t)(t - 1) * count] = r;
        else TG_CHECK_LOW(st.qp, rowS<B>(j));
    }
    if (TG_CHECK_ENABLED) {
        // the window of Lw+1 limbs holds y_k mod 2^(32 (Lw+1)): a negative y_k
        // adds -A_jk 2^(32 (Lw+1)) to the dividend (csrc/check.cuh)
        uint64_t corr = 0;
#pragma unroll
        for (int k = 0; k < NP; ++k) corr += (uint64_t)rowA<B>(j, k) * (fill[k] & 1u);
        TG_CHECK_END(st.acc - corr, st.bor, rowO<B>(j));
    }
}

}  // namespace tg
