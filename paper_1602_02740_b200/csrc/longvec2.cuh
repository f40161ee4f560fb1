// Two-pass long-vector op executor (replaces the single-pass decoupled
// look-back of longvec.cuh for the upper levels of C4/C5).
//
// An op  dst = ((sum_i m_i (S_i << s_i)) / o) >> shr  over W limbs is run as
//   pass 1  (k_lop2 / k_lmulti2, phase 1): every tile (NT threads x CH limbs)
//           forms its linear combination lin_p (64/128-bit) and publishes a
//           SUMMARY: its carry map (the signed carry out of the tile as a
//           3-piece function of the carry in, as in longvec.cuh) and its
//           residue  l'_k = sum_{p in tile} lin_p 2^(32 (p - t0)) mod o;
//   scan    (k_lscan2): one warp per (instance, output) turns the summaries
//           into every tile's carry-in c_t0 and 2-adic borrow-in beta_t0;
//   (phase 3: an instance that fits one tile skips pass 1 and the scan)
//   pass 2  (phase 2): every tile recomputes lin_p, resolves its threads'
//           carry-ins with a warp scan of the thread carry maps, their borrow-
//           ins from the closed form below, and writes the exact quotient
//           limbs, shifted.
// No tile ever waits for another (the look-back chains of the single-pass
// executor were the bottleneck: 25% warps active, 7-8 barrier stalls per
// issue in the ncu full set of an earlier session of round 2; round 1 counters: profiles/r01_c4_launches_summary.txt).
//
// The borrow of the exact division never needs the normalised limbs of the
// predecessors: with L_p = sum_{i<p} lin_i 2^(32 i) (unnormalised) and c_p the
// carry into position p,  X mod 2^(32p) = L_p - c_p 2^(32p),  so the borrow
// closed form beta_p = -(X mod 2^(32p)) 2^(-32p) mod o is
//     beta_p = (c_p - B_p) mod o,    B_p = 2^(-32p) L_p mod o,
// and B obeys the affine recurrence B_{t0+TL} = (B_t0 + l'_k) M^-1 with
// M = 2^(32 TL) mod o: residues are additive, carries are a separate scan.
#pragma once

namespace tg {

// per-tile record: pass-1 summary, then the scan's carry-in / borrow-in
struct LTile {
    long long lo, hi;          // piece thresholds of the tile's carry map
    long long cout[3];         // carry out for piece 0 / 1 / 2 of the carry in
    uint32_t ell;              // l'_k (tile-relative residue of lin), mod o
    uint32_t beta;             // borrow into the tile (scan output)
    long long cin;             // carry into the tile (scan output)
};

struct LCMap {                 // carry map c -> cout[piece(c)]
    long long lo, hi, cout[3];
};
__device__ __forceinline__ int lc_piece(const LCMap& A, long long c) { return c < A.lo ? 0 : (c >= A.hi ? 2 : 1); }
__device__ __forceinline__ long long lc_apply(const LCMap& A, long long c) { return lv_sel(A.cout, lc_piece(A, c)); }
// A then B
__device__ __forceinline__ LCMap lc_compose(const LCMap& A, const LCMap& B) {
    LCMap C;
    C.lo = A.lo;
    C.hi = A.hi;
#pragma unroll
    for (int p = 0; p < 3; ++p) C.cout[p] = lc_apply(B, A.cout[p]);
    return C;
}
__device__ __forceinline__ LCMap lc_identity() {
    LCMap I;
    I.lo = LLONG_MIN;   // piece 1 for every c: identity needs cout = c, which a
    I.hi = LLONG_MAX;   // 3-piece constant map cannot express -> flag below
    I.cout[0] = I.cout[1] = I.cout[2] = 0;
    return I;
}
__device__ __forceinline__ LCMap lc_shfl_up(const LCMap& a, int d) {
    LCMap r;
    r.lo = __shfl_up_sync(0xffffffffu, a.lo, d);
    r.hi = __shfl_up_sync(0xffffffffu, a.hi, d);
#pragma unroll
    for (int p = 0; p < 3; ++p) r.cout[p] = __shfl_up_sync(0xffffffffu, a.cout[p], d);
    return r;
}

// (c mod o) for a signed 64-bit c
__device__ __forceinline__ uint32_t lv2_modc(long long c, const LMod& M) {
    const uint32_t r = lv_mod((unsigned long long)(c < 0 ? -c : c), M);
    return (c < 0 && r) ? M.o - r : r;
}
__device__ __forceinline__ uint32_t lv2_addmod(uint32_t a, uint32_t b, uint32_t o) {
    const uint32_t s = a + b;
    return (s < a || s >= o) ? s - o : s;
}
__device__ __forceinline__ uint32_t lv2_powmod(uint32_t b, unsigned e, const LMod& M) {
    uint32_t r = 1u % M.o;
    while (e) {
        if (e & 1u) r = lv_mulmod(r, b, M);
        b = lv_mulmod(b, b, M);
        e >>= 1;
    }
    return r;
}

// words of the padded quotient buffer (TL + halo positions, one pad per CH)
__host__ __device__ inline int lv2_qwords(int TL, int CH) {
    return TL + LV_MAXHALO + 1 + (TL + LV_MAXHALO + 1) / CH + 1;
}
inline size_t lop2_smem(int nthreads, int ch) {
    return 4 * ((size_t)lv2_qwords(nthreads * ch, ch) + (size_t)(ch + 1) * (nthreads + 1));
}
inline size_t lmulti2_smem(int nthreads, int ch, int ns) {
    const int np1 = nthreads + 1 + (LM_HALO + ch - 1) / ch;
    return 4 * ((size_t)lv2_qwords(nthreads * ch, ch) + (size_t)ns * ch * np1);
}

struct L2Smem {
    LCMap wmap[LV_NT / 32];    // warp carry maps (inclusive of the whole warp)
    uint32_t wres[LV_NT / 32]; // warp residue sums (weighted, tile-relative)
    uint32_t mw32;             // Mch^32 mod o
};

// Pass 1 / pass 2 of one output of one tile.  lin: this thread's CH
// positions p0 = tstart + tid*CH.  P.st_base + tile*st_stride is the tile's
// LTile record.
// sum of v over the lanes of a warp (every lane gets it)
__device__ __forceinline__ long long lv2_warp_sum(long long v) {
#pragma unroll
    for (int d = 16; d; d >>= 1) v += __shfl_xor_sync(0xffffffffu, v, d);
    return v;
}
__device__ __forceinline__ __int128 lv2_warp_sum(__int128 v) {
    unsigned long long lo = (unsigned long long)v;
    long long hi = (long long)(v >> 64);
#pragma unroll
    for (int d = 16; d; d >>= 1) {
        const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, d);
        const long long h2 = __shfl_xor_sync(0xffffffffu, hi, d);
        const unsigned long long sl = lo + l2;
        hi += h2 + (sl < lo ? 1 : 0);
        lo = sl;
    }
    return ((__int128)hi << 64) | (__int128)lo;
}

// COOP: halo_fn(h, lane) is lane's share of the terms of halo position h,
// summed over the last warp (the halo of a multi-output op, a serial loop
// over every term on one thread otherwise, was the tail of pass 2:
// profiles/r02_c5top_*); else halo_fn(hl) fills all positions on one thread.
template <typename Acc, int CH, bool COOP = false, class HaloF>
__device__ __forceinline__ void lv2_tile(const Acc (&lin)[CH], const LMod& M, const LFinish& P, unsigned tile,
                                         int tstart, L2Smem& sh, uint32_t* Q, HaloF halo_fn, int phase) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int NT = blockDim.x, NW = NT >> 5, TL = NT * CH;
    const uint32_t o = M.o;
    LTile* T = reinterpret_cast<LTile*>(P.st_base) + (long long)tile * P.st_stride;
    // local normalisation (carry-in 0) -> this thread's carry map
    uint32_t x[CH];
    long long c = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const Acc v = lin[q] + (Acc)c;
        x[q] = (uint32_t)v;
        c = (long long)(v >> 32);
    }
    LCMap A;
    {
        const unsigned long long L64 = (unsigned long long)x[0] | ((unsigned long long)x[1] << 32);
        bool tz = true, to = true;
#pragma unroll
        for (int q = 2; q < CH; ++q) { tz &= (x[q] == 0u); to &= (x[q] == 0xFFFFFFFFu); }
        A.lo = (tz && L64 <= 0x8000000000000000ull) ? (long long)(0ull - L64) : LLONG_MIN;
        const unsigned long long comp = 0ull - L64;
        A.hi = (to && L64 != 0 && comp <= (unsigned long long)LLONG_MAX) ? (long long)comp : LLONG_MAX;
        A.cout[0] = c - 1;
        A.cout[1] = c;
        A.cout[2] = c + 1;
    }
    // weighted residue of this thread's positions: s = Mch^tid (x + c 2^(32 CH)) mod o
    uint32_t s = 0, wt = 1, wti = 1;
    if (o > 1) {
        uint32_t r = 0;
#pragma unroll
        for (int q = CH - 1; q >= 0; --q) r = lv_mod((unsigned long long)r * P.p32 + x[q], M);
        r = lv2_addmod(r, lv_mulmod(lv2_modc(c, M), P.Mch, M), o);
        // Mch^lane by a warp product scan, times (Mch^32)^warp
        uint32_t pw = P.Mch;   // inclusive scan of Mch over lanes -> Mch^(lane+1)
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const uint32_t t = __shfl_up_sync(0xffffffffu, pw, d);
            if (lane >= d) pw = lv_mulmod(pw, t, M);
        }
        const uint32_t m32 = __shfl_sync(0xffffffffu, pw, 31);   // Mch^32
        pw = __shfl_up_sync(0xffffffffu, pw, 1);
        if (lane == 0) pw = 1u % o;                              // Mch^lane
        uint32_t wb = 1u % o;
        for (int w = 0; w < warp; ++w) wb = lv_mulmod(wb, m32, M);
        wt = lv_mulmod(pw, wb, M);                               // Mch^tid
        s = lv_mulmod(r, wt, M);
        if (phase >= 2) {
            // inverse weight mi^tid (mi = Mch^-1)
            uint32_t pi = P.mi;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const uint32_t t = __shfl_up_sync(0xffffffffu, pi, d);
                if (lane >= d) pi = lv_mulmod(pi, t, M);
            }
            const uint32_t mi32 = __shfl_sync(0xffffffffu, pi, 31);
            pi = __shfl_up_sync(0xffffffffu, pi, 1);
            if (lane == 0) pi = 1u % o;
            uint32_t wbi = 1u % o;
            for (int w = 0; w < warp; ++w) wbi = lv_mulmod(wbi, mi32, M);
            wti = lv_mulmod(pi, wbi, M);
        }
    }
    // warp inclusive scans: carry maps (composition) and residues (sum)
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
    if (lane == 31) {
        sh.wmap[warp] = inc;
        sh.wres[warp] = sinc;
    }
    __syncthreads();
    if (phase == 1) {
        if (tid == 0) {
            LCMap Tm = sh.wmap[0];
            uint32_t ell = sh.wres[0];
            for (int w = 1; w < NW; ++w) {
                Tm = lc_compose(Tm, sh.wmap[w]);
                if (o > 1) ell = lv2_addmod(ell, sh.wres[w], o);
            }
            T->lo = Tm.lo;
            T->hi = Tm.hi;
            T->cout[0] = Tm.cout[0];
            T->cout[1] = Tm.cout[1];
            T->cout[2] = Tm.cout[2];
            T->ell = o > 1 ? ell : 0u;
        }
        return;
    }
    // ---- pass 2: this thread's carry-in and borrow-in
    const LCMap excl = lc_shfl_up(inc, 1);          // valid for lane > 0
    const uint32_t sexcl = __shfl_up_sync(0xffffffffu, sinc, 1);
    long long cin = phase == 3 ? 0 : T->cin;       // phase 3: the tile is the whole vector
    const uint32_t tb = phase == 3 ? 0u : T->beta;
    uint32_t Bt = 0;                                 // B at the tile start
    if (o > 1) Bt = lv2_addmod(lv2_modc(cin, M), tb ? o - tb : 0u, o);   // beta_t0 = c_t0 - B_t0
    uint32_t lam = 0;                                // weighted residues of the threads before this one
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
        // beta_p0 = c_p0 - Mch^-tid (B_t0 + Lambda) mod o
        const uint32_t bp = lv_mulmod(lv2_addmod(Bt, lam, o), wti, M);
        beta = lv2_addmod(lv2_modc(cin, M), bp ? o - bp : 0u, o);
    }
    // exact limbs, exact division, quotients to smem
    c = cin;
#pragma unroll
    for (int q = 0; q < CH; ++q) {
        const Acc v = lin[q] + (Acc)c;
        uint32_t xq = (uint32_t)v;
        c = (long long)(v >> 32);
        if (o > 1) xq = tg_divexact_step(xq, beta, P.oinv, o);
        Q[tid * (CH + 1) + q] = xq;   // padded: conflict-free (position i at i + i / CH)
    }
    const int halo = P.sa + (P.sr ? 1 : 0);
    if constexpr (COOP) {
        if (warp == NW - 1) {
#pragma unroll 1
            for (int h = 0; h < halo; ++h) {
                const Acc v = lv2_warp_sum(halo_fn(h, lane)) + (Acc)c;   // (c, beta: lane 31's, the tile's last thread)
                if (lane == 31) {
                    uint32_t xq = (uint32_t)v;
                    c = (long long)(v >> 32);
                    if (o > 1) xq = tg_divexact_step(xq, beta, P.oinv, o);
                    Q[TL + h + (TL + h) / CH] = xq;
                }
            }
        }
    } else {
        if (tid == NT - 1 && halo > 0) {
            Acc hl[LV_MAXHALO];
            halo_fn(hl);
#pragma unroll
            for (int h = 0; h < LV_MAXHALO; ++h) {
                if (h >= halo) break;
                const Acc v = hl[h] + (Acc)c;
                uint32_t xq = (uint32_t)v;
                c = (long long)(v >> 32);
                if (o > 1) xq = tg_divexact_step(xq, beta, P.oinv, o);
                Q[TL + h + (TL + h) / CH] = xq;
            }
        }
    }
    __syncthreads();
    uint32_t* dst = P.dst;
    for (int i = tid; i < TL; i += NT) {
        const int t = tstart + i;
        if (t >= P.W) break;
        const int i0 = i + P.sa, i1 = i0 + 1;
        const uint32_t lo = Q[i0 + i0 / CH];
        const uint32_t y = P.sr ? __funnelshift_r(lo, Q[i1 + i1 / CH], P.sr) : lo;
        dst[(long long)t * P.dst_limb_stride] = y;
    }
}

// linear combination of one tile of a single-output op (the term slices staged
// through shared memory, as k_long_op)
template <typename Acc, int CH>
__device__ __forceinline__ void lop2_lincomb(const LOpDev& op, long long inst, int tstart, uint32_t* Sx, Acc (&lin)[CH]) {
    const int tid = threadIdx.x, NT = blockDim.x, TL = NT * CH, NP1 = NT + 1;
    Acc cst = 0;
#pragma unroll
    for (int q = 0; q < CH; ++q) lin[q] = 0;
    for (int kk = 0; kk < op.nt; ++kk) {
        const LTermDev& T = op.t[kk];
        const int ilo = tstart - T.a - 1, ihi = tstart + TL - 1 - T.a;
        if (ihi < 0) continue;
        const uint32_t* src = T.base + inst * T.inst_stride;
        uint32_t fill = 0;
        if (T.sign && T.len > 0) fill = (__ldg(src + (long long)(T.len - 1) * T.limb_stride) >> 31) ? 0xFFFFFFFFu : 0u;
        if (ilo >= T.len) {
            cst += (Acc)T.m * (Acc)fill;
            continue;
        }
        __syncthreads();
        {
            uint32_t xv[CH];
            if (ilo + 1 >= 0 && ihi < T.len) {
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
                const int idx = ilo;
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
        uint32_t prev = tid ? Sx[(CH - 1) * NP1 + tid - 1] : Sx[CH * NP1];
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const uint32_t cur = Sx[q * NP1 + tid];
            const uint32_t xx = r ? __funnelshift_l(prev, cur, r) : cur;
            lin[q] += (Acc)m * (Acc)xx;
            prev = cur;
        }
    }
#pragma unroll
    for (int q = 0; q < CH; ++q) lin[q] += cst;
    __syncthreads();
}

template <bool WIDE, int CH>
__global__ void __launch_bounds__(LV_NT, WIDE ? 2 : 3) k_lop2(const LOpDev* __restrict__ opp, LTile* __restrict__ tiles, int phase) {
    using Acc = typename std::conditional<WIDE, __int128, long long>::type;
    __shared__ __align__(16) LOpDev s_op;
    {
        const int4* srcd = reinterpret_cast<const int4*>(opp);
        int4* dstd = reinterpret_cast<int4*>(&s_op);
        constexpr int NQ = (int)(sizeof(LOpDev) / 16);
        for (int i = threadIdx.x; i < NQ; i += blockDim.x) dstd[i] = __ldg(srcd + i);
    }
    __shared__ L2Smem s_sh;
    extern __shared__ uint32_t Q[];
    __syncthreads();
    const LOpDev& op = s_op;
    const unsigned tile = blockIdx.x;
    const long long inst = tile / op.tiles_per_inst;
    const int k = (int)(tile - inst * op.tiles_per_inst);
    const int TL = blockDim.x * CH;
    const int tstart = k * TL;
    const LMod M{op.o, op.orcp};
    Acc lin[CH];
    lop2_lincomb<Acc, CH>(op, inst, tstart, Q + lv2_qwords(TL, CH), lin);
    lv2_tile<Acc, CH>(lin, M,
                      LFinish{op.oinv, op.p32, op.Mch, op.mi, op.sa, op.sr, op.W, reinterpret_cast<LStatus*>(tiles), 1,
                              op.dst + inst * op.dst_inst_stride, op.dst_limb_stride},
                      tile, tstart, s_sh, Q,
                      [&](Acc (&hl)[LV_MAXHALO]) { lv_lincomb<Acc, LV_MAXHALO>(op, op.nt, inst, tstart + TL, hl); }, phase);
}

// multi-output op: sources staged once per tile, every output in turn
template <bool WIDE, int CH>
__global__ void __launch_bounds__(LV_NT, WIDE ? 2 : 3) k_lmulti2(const LMultiDev* __restrict__ dp, LTile* __restrict__ tiles,
                                                      int phase) {
    using Acc = typename std::conditional<WIDE, __int128, long long>::type;
    __shared__ __align__(16) LMultiDev s_d;
    {
        const int4* srcd = reinterpret_cast<const int4*>(dp);
        int4* dstd = reinterpret_cast<int4*>(&s_d);
        constexpr int NQ = (int)(sizeof(LMultiDev) / 16);
        for (int i = threadIdx.x; i < NQ; i += blockDim.x) dstd[i] = __ldg(srcd + i);
    }
    __shared__ L2Smem s_sh;
    extern __shared__ uint32_t dsm[];
    __syncthreads();
    const int tid = threadIdx.x, NT = blockDim.x, TL = NT * CH, NP1 = NT + 1 + (LM_HALO + CH - 1) / CH;
    uint32_t* Q = dsm;
    uint32_t* Sb = dsm + lv2_qwords(TL, CH);
    const LMultiDev& d = s_d;
    const unsigned tile = blockIdx.x;
    const long long inst = tile / d.tiles_per_inst;
    const int kt = (int)(tile - inst * d.tiles_per_inst);
    const int tstart = kt * TL;
    for (int sI = 0; sI < d.ns; ++sI) {
        const LMSrc& S = d.src[sI];
        const uint32_t* sp = S.base + inst * S.is;
        uint32_t fill = 0;
        if (S.sign && S.len > 0) fill = (__ldg(sp + (S.len - 1)) >> 31) ? 0xFFFFFFFFu : 0u;
        uint32_t* sj = Sb + (size_t)sI * CH * NP1;
        // all loads of a thread before its stores (TL = NT * CH)
        uint32_t xv[CH];
        if (tstart + TL <= S.len) {
#pragma unroll
            for (int q = 0; q < CH; ++q) xv[q] = __ldg(sp + tstart + tid + q * NT);
        } else {
#pragma unroll
            for (int q = 0; q < CH; ++q) {
                const int t = tstart + tid + q * NT;
                xv[q] = (t < S.len) ? __ldg(sp + t) : fill;
            }
        }
#pragma unroll
        for (int q = 0; q < CH; ++q) {
            const int i = tid + q * NT;
            sj[(i % CH) * NP1 + i / CH] = xv[q];
        }
        if (tid < LM_HALO) {
            const int i = TL + tid, t = tstart + i;
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
        lv2_tile<Acc, CH, true>(lin, M,
                          LFinish{O.oinv, O.p32, O.Mch, O.mi, O.sa, O.sr, d.W,
                                  reinterpret_cast<LStatus*>(tiles + o), d.no, O.dst + inst * d.dst_is, d.dst_ls},
                          tile, tstart, s_sh, Q,
                          [&](int h, int part) -> Acc {   // lane `part`: the sources s2 = part (mod 32)
                              Acc v = 0;
                              const int i = TL + h;
                              for (int s2 = part; s2 < d.ns; s2 += 32)
                                  v += (Acc)d.m[o][s2] * (Acc)Sb[(size_t)s2 * CH * NP1 + (i % CH) * NP1 + i / CH];
                              return v;
                          },
                          phase);
        __syncthreads();   // Q / s_sh reuse by the next output
    }
}

// scan: one warp per (instance, output).  Tile records of (instance i,
// output o) at tiles[(i*tpi + k)*no + o].  Lane L owns tiles [L r, L r + r).
struct L2ScanArgs {
    LTile* tiles;
    int count, tpi, no, nthreads, ch;
    uint32_t o[LM_MAXO];
    unsigned long long orcp[LM_MAXO];
    uint32_t mch[LM_MAXO], mi[LM_MAXO];   // 2^(32 CH) mod o and its inverse
};

// the same scan with one 1024-thread CTA per (instance, output), for vectors
// of many tiles (the T16 top level of C5: 513 tiles; a single warp walking
// 17 tiles per lane measured 25 us per op, the latency of its serial runs)
__global__ void __launch_bounds__(1024) k_lscan2_blk(L2ScanArgs A) {
    const int gw = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
    const int inst = gw / A.no, oi = gw - inst * A.no;
    const uint32_t o = A.o[oi];
    const LMod M{o, A.orcp[oi]};
    const uint32_t Minv = o > 1 ? lv2_powmod(A.mi[oi], (unsigned)A.nthreads, M) : 0u;
    const int T = A.tpi, r = (T + blockDim.x - 1) / blockDim.x;
    const int k0 = min(tid * r, T), k1 = min(k0 + r, T);
    LTile* base = A.tiles + (long long)inst * T * A.no + oi;
    bool has = false;
    LCMap cm = lc_identity();
    uint32_t a = 1u % (o ? o : 1u), g = 0;
    for (int k = k0; k < k1; ++k) {
        const LTile& t = base[(long long)k * A.no];
        LCMap x;
        x.lo = t.lo; x.hi = t.hi; x.cout[0] = t.cout[0]; x.cout[1] = t.cout[1]; x.cout[2] = t.cout[2];
        cm = has ? lc_compose(cm, x) : x;
        has = true;
        if (o > 1) {
            a = lv_mulmod(a, Minv, M);
            g = lv_mulmod(lv2_addmod(g, t.ell, o), Minv, M);
        }
    }
    bool ihas = has;
    LCMap icm = cm;
    uint32_t ia = a, ig = g;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const LCMap pm = lc_shfl_up(icm, d);
        const bool ph = __shfl_up_sync(0xffffffffu, ihas, d);
        const uint32_t pa = __shfl_up_sync(0xffffffffu, ia, d), pg = __shfl_up_sync(0xffffffffu, ig, d);
        if (lane >= d && ph) {
            icm = ihas ? lc_compose(pm, icm) : pm;
            if (o > 1) {
                ig = lv2_addmod(lv_mulmod(pg, ia, M), ig, o);
                ia = lv_mulmod(pa, ia, M);
            }
            ihas = true;
        }
    }
    __shared__ LCMap wcm[32];
    __shared__ uint32_t wa[32], wg[32];
    __shared__ bool wh[32];
    __shared__ long long wc_in[32];
    __shared__ uint32_t wB_in[32];
    if (lane == 31) { wcm[warp] = icm; wa[warp] = ia; wg[warp] = ig; wh[warp] = ihas; }
    __syncthreads();
    if (tid == 0) {   // states at the start of every warp's runs (instance start: c = 0, B = 0)
        long long c = 0;
        uint32_t B = 0;
        for (int w = 0; w < NW; ++w) {
            wc_in[w] = c;
            wB_in[w] = B;
            if (wh[w]) {
                c = lc_apply(wcm[w], c);
                if (o > 1) B = lv2_addmod(lv_mulmod(B, wa[w], M), wg[w], o);
            }
        }
    }
    __syncthreads();
    const LCMap em = lc_shfl_up(icm, 1);
    const bool eh = __shfl_up_sync(0xffffffffu, ihas, 1) && lane > 0;
    const uint32_t ea = __shfl_up_sync(0xffffffffu, ia, 1), eg = __shfl_up_sync(0xffffffffu, ig, 1);
    long long c = wc_in[warp];
    uint32_t B = wB_in[warp];
    if (eh) {
        c = lc_apply(em, c);
        if (o > 1) B = lv2_addmod(lv_mulmod(B, ea, M), eg, o);
    }
    for (int k = k0; k < k1; ++k) {
        LTile& t = base[(long long)k * A.no];
        t.cin = c;
        t.beta = o > 1 ? lv2_addmod(lv2_modc(c, M), B ? o - B : 0u, o) : 0u;
        LCMap x;
        x.lo = t.lo; x.hi = t.hi; x.cout[0] = t.cout[0]; x.cout[1] = t.cout[1]; x.cout[2] = t.cout[2];
        c = lc_apply(x, c);
        if (o > 1) B = lv_mulmod(lv2_addmod(B, t.ell, o), Minv, M);
    }
}

__global__ void __launch_bounds__(256) k_lscan2(L2ScanArgs A) {
    const int gw = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5);
    const int lane = threadIdx.x & 31;
    if (gw >= A.count * A.no) return;
    const int inst = gw / A.no, oi = gw - inst * A.no;
    const uint32_t o = A.o[oi];
    const LMod M{o, A.orcp[oi]};
    // M^-1 = (Mch^-1)^NT
    const uint32_t Minv = o > 1 ? lv2_powmod(A.mi[oi], (unsigned)A.nthreads, M) : 0u;
    const int T = A.tpi, r = (T + 31) / 32;
    const int k0 = min(lane * r, T), k1 = min(k0 + r, T);
    LTile* base = A.tiles + (long long)inst * T * A.no + oi;
    // run aggregates: carry map and the affine residue map B -> B a + g
    bool has = false;
    LCMap cm = lc_identity();
    uint32_t a = 1u % (o ? o : 1u), g = 0;
    for (int k = k0; k < k1; ++k) {
        const LTile& t = base[(long long)k * A.no];
        LCMap x;
        x.lo = t.lo; x.hi = t.hi; x.cout[0] = t.cout[0]; x.cout[1] = t.cout[1]; x.cout[2] = t.cout[2];
        cm = has ? lc_compose(cm, x) : x;
        has = true;
        if (o > 1) {   // B' = (B + l) Minv
            a = lv_mulmod(a, Minv, M);
            g = lv_mulmod(lv2_addmod(g, t.ell, o), Minv, M);
        }
    }
    // warp exclusive scan of (has, carry map, affine map), composed in lane order
    bool ihas = has;
    LCMap icm = cm;
    uint32_t ia = a, ig = g;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        const LCMap pm = lc_shfl_up(icm, d);
        const bool ph = __shfl_up_sync(0xffffffffu, ihas, d);
        const uint32_t pa = __shfl_up_sync(0xffffffffu, ia, d), pg = __shfl_up_sync(0xffffffffu, ig, d);
        if (lane >= d && ph) {
            icm = ihas ? lc_compose(pm, icm) : pm;
            if (o > 1) {   // prev then mine: x -> (x pa + pg) ia + ig
                ig = lv2_addmod(lv_mulmod(pg, ia, M), ig, o);
                ia = lv_mulmod(pa, ia, M);
            }
            ihas = true;
        }
    }
    // exclusive: apply the inclusive state of lane-1 to the instance start (c = 0, B = 0)
    const LCMap em = lc_shfl_up(icm, 1);
    const bool eh = __shfl_up_sync(0xffffffffu, ihas, 1) && lane > 0;
    const uint32_t eg = __shfl_up_sync(0xffffffffu, ig, 1);
    long long c = eh ? lc_apply(em, 0) : 0;
    uint32_t B = (eh && o > 1) ? eg : 0u;   // B0 = 0: B = 0 * a + g
    for (int k = k0; k < k1; ++k) {
        LTile& t = base[(long long)k * A.no];
        t.cin = c;
        t.beta = o > 1 ? lv2_addmod(lv2_modc(c, M), B ? o - B : 0u, o) : 0u;
        LCMap x;
        x.lo = t.lo; x.hi = t.hi; x.cout[0] = t.cout[0]; x.cout[1] = t.cout[1]; x.cout[2] = t.cout[2];
        c = lc_apply(x, c);
        if (o > 1) B = lv_mulmod(lv2_addmod(B, t.ell, o), Minv, M);
    }
}

}  // namespace tg

namespace tg {
// ------------------------------------------------------------------------
// Multi-output op with WIDE multipliers (the matrix-form Toom-16
// interpolation): out_o = ((sum_s m_os src_s) / o_o) >> shr_o
// with m_os = sum_d a_osd 2^(32 d) given as balanced 32-bit digits, so a
// position p of the linear combination is sum_s sum_d a_osd src_s[p - d]
// (int64 products, int128 accumulation).  Sources are staged once per tile
// with LB_PRE limbs before the tile; the scans are those of k_lmulti2.
// ------------------------------------------------------------------------
constexpr int LB_MAXS = 17, LB_MAXO = 15, LB_ND = 4, LB_PRE = LB_ND - 1, LB_CH = 8;

struct __align__(16) LBigDev {
    int ns, no, W, tiles_per_inst, nthreads, ch, count, pad;
    long long dst_is, dst_ls;
    LMSrc src[LB_MAXS];
    LMOut out[LB_MAXO];
    int nd[LB_MAXO][LB_MAXS];          // digits in use (0: the source is not a term)
    int a[LB_MAXO][LB_MAXS][LB_ND];
};

__host__ __device__ inline int lbig2_np1(int nthreads) { return nthreads + (LB_PRE + LM_HALO + LB_CH - 1) / LB_CH + 1; }
inline size_t lbig2_smem(int nthreads, int ns) {
    return 4 * ((size_t)lv2_qwords(nthreads * LB_CH, LB_CH) + (size_t)ns * LB_CH * lbig2_np1(nthreads));
}

__global__ void __launch_bounds__(128, 3) k_lbig2(const LBigDev* __restrict__ dp, LTile* __restrict__ tiles, int phase) {
    constexpr int CH = LB_CH;
    using Acc = __int128;
    __shared__ __align__(16) LBigDev s_d;
    {
        const int4* srcd = reinterpret_cast<const int4*>(dp);
        int4* dstd = reinterpret_cast<int4*>(&s_d);
        constexpr int NQ = (int)(sizeof(LBigDev) / 16);
        for (int i = threadIdx.x; i < NQ; i += blockDim.x) dstd[i] = __ldg(srcd + i);
    }
    __shared__ L2Smem s_sh;
    extern __shared__ uint32_t dsm[];
    __syncthreads();
    const int tid = threadIdx.x, NT = blockDim.x, TL = NT * CH, NP1 = lbig2_np1(NT);
    uint32_t* Q = dsm;
    uint32_t* Sb = dsm + lv2_qwords(TL, CH);   // [ns][CH][NP1]: relative position i = pos - tstart + LB_PRE
    const LBigDev& d = s_d;
    const unsigned tile = blockIdx.x;
    const long long inst = tile / d.tiles_per_inst;
    const int kt = (int)(tile - inst * d.tiles_per_inst);
    const int tstart = kt * TL;
    // staging: every thread issues the loads of two sources before storing
    // (a load-store loop per element was latency-bound: 11 long-scoreboard
    // stalls per issue, ncu full set of an earlier session; the current counters: profiles/r02_c5top_*)
    constexpr int EX = (LB_PRE + LM_HALO + 31) / 32;   // extra elements past TL, per warp lane
    for (int s0 = 0; s0 < d.ns; s0 += 2) {
        uint32_t xv[2][CH + EX];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int sI = s0 + h;
            if (sI >= d.ns) break;
            const LMSrc& S = d.src[sI];
            const uint32_t* sp = S.base + inst * S.is;
            uint32_t fill = 0;
            if (S.sign && S.len > 0) fill = (__ldg(sp + (S.len - 1)) >> 31) ? 0xFFFFFFFFu : 0u;
#pragma unroll
            for (int q = 0; q < CH + EX; ++q) {
                const int i = tid + q * NT;   // relative index; q >= CH: the tail past TL
                const int t = tstart - LB_PRE + i;
                xv[h][q] = (q >= CH && i >= TL + LB_PRE + LM_HALO) ? 0u
                           : (t < 0 ? 0u : (t < S.len ? __ldg(sp + t) : fill));
            }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int sI = s0 + h;
            if (sI >= d.ns) break;
            uint32_t* sj = Sb + (size_t)sI * CH * NP1;
#pragma unroll
            for (int q = 0; q < CH + EX; ++q) {
                const int i = tid + q * NT;
                if (q < CH || i < TL + LB_PRE + LM_HALO) sj[(i % CH) * NP1 + i / CH] = xv[h][q];
            }
        }
    }
    __syncthreads();
    auto staged = [&](int sI, int i) -> uint32_t { return Sb[(size_t)sI * CH * NP1 + (i % CH) * NP1 + i / CH]; };
    static_assert(LB_PRE == LB_ND - 1, "the window of a thread starts LB_ND - 1 positions early");
    for (int o = 0; o < d.no; ++o) {
        const LMOut& O = d.out[o];
        // each balanced 32-bit digit a = h 2^16 + l (0 <= l < 2^16) enters as
        // two IMAD.WIDE.U32 terms into 64-bit sums of < 2^48 terms (no
        // overflow for <= 2^16 terms): P0 = sum l y, P1 - N1 = sum h y, then
        // lin = P0 + (P1 - N1) 2^16 (int128 once per output)
        uint64_t P0[CH], P1[CH], N1[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) P0[q] = P1[q] = N1[q] = 0ull;
        for (int sI = 0; sI < d.ns; ++sI) {
            const int nd = d.nd[o][sI];
            // the source window of this thread: relative indices tid*CH + q', q' < CH + LB_PRE
            uint32_t yw[CH + LB_PRE];
            const uint32_t* sb = Sb + (size_t)sI * CH * NP1 + tid;
#pragma unroll
            for (int q = 0; q < CH + LB_PRE; ++q) yw[q] = sb[(q % CH) * NP1 + q / CH];
#pragma unroll
            for (int dd = 0; dd < LB_ND; ++dd) {
                if (dd >= nd) break;
                const long long a = d.a[o][sI][dd];
                if (a == 0) continue;
                const uint32_t l = (uint32_t)a & 0xFFFFu;
                const long long h = (a - (long long)l) >> 16;
                // position p0 + q - dd  ->  window index q - dd + LB_PRE
#pragma unroll
                for (int q = 0; q < CH; ++q) P0[q] = tg_madw(l, yw[q - dd + LB_PRE], P0[q]);
                if (h > 0) {
#pragma unroll
                    for (int q = 0; q < CH; ++q) P1[q] = tg_madw((uint32_t)h, yw[q - dd + LB_PRE], P1[q]);
                } else if (h < 0) {
#pragma unroll
                    for (int q = 0; q < CH; ++q) N1[q] = tg_madw((uint32_t)(-h), yw[q - dd + LB_PRE], N1[q]);
                }
            }
        }
        Acc lin[CH];
#pragma unroll
        for (int q = 0; q < CH; ++q) lin[q] = (Acc)P0[q] + ((Acc)(long long)(P1[q] - N1[q]) << 16);
        const LMod M{O.o, O.orcp};
        lv2_tile<Acc, CH, true>(lin, M,
                          LFinish{O.oinv, O.p32, O.Mch, O.mi, O.sa, O.sr, d.W,
                                  reinterpret_cast<LStatus*>(tiles + o), d.no, O.dst + inst * d.dst_is, d.dst_ls},
                          tile, tstart, s_sh, Q,
                          [&](int h, int part) -> Acc {   // lane `part`: the sources s2 = part (mod 32)
                              Acc v = 0;
                              for (int s2 = part; s2 < d.ns; s2 += 32)
                                  for (int dd = 0; dd < d.nd[o][s2]; ++dd)
                                      v += (Acc)((long long)d.a[o][s2][dd] * (long long)staged(s2, TL + h - dd + LB_PRE));
                              return v;
                          },
                          phase);
        __syncthreads();
    }
}
}  // namespace tg
