/*
 * libtoomgpu -- B200-native (sm_100a) batched B-way Toom-Cook multiplication.
 *
 * The operation (§1, Eqs. 1.1-1.3): for unsigned integers u,
 * v split into B blocks of b bits, u = U(2^b), v = V(2^b), compute
 * w = u*v = W(2^b) by (1) evaluating U and V at 2B-1 small points,
 * (2) forming the 2B-1 products y_k = U(x_k) V(x_k) recursively
 * (Eq. 2.1; "lower-level products can also be done in parallel"),
 * (3) interpolating W's coefficients with the even-odd method (§4,
 * Eqs. 4.5-4.6) and the Newton listings with exact divisions (§3,
 * PAPER.md:114-120, 154-158), (4) recomposing w = W(2^b) with carries.
 *
 * Conventions for every entry point:
 *   - limbs are uint32_t, little-endian (the paper's 32-bit words);
 *   - unless a name ends in _host, every pointer is a DEVICE pointer owned by
 *     the caller; the library never frees caller memory;
 *   - calls are asynchronous and ordered on `stream` (a cudaStream_t, NULL =
 *     legacy default stream); argument errors return immediately, before any
 *     work is enqueued;
 *   - w must not overlap u or v (TOOM_EINVAL);
 *   - the output is fixed length (nu+nv, or 2n per batched product), high
 *     limbs zero, not normalized;
 *   - no exceptions cross the ABI; all functions are thread-compatible
 *     (one stream per host thread), not re-entrant on one stream.
 *
 * There is no CPU fallback: without a usable sm_100 device every compute
 * entry point returns TOOM_ECUDA.
 */
#ifndef TOOMGPU_H
#define TOOMGPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    TOOM_OK = 0,
    TOOM_EINVAL = 1,       /* bad argument (null pointer, aliasing, unsupported B, size) */
    TOOM_EVERIFY = 2,      /* result verification failed (residue check, toom_set_verify) */
    TOOM_EINEXACT = 3,     /* an exact division was not exact (exit code 3) */
    TOOM_ENOMEM = 4,       /* device workspace allocation failed */
    TOOM_ECUDA = 5,        /* a CUDA runtime error (no device, launch failure, ...) */
    TOOM_EUNSUPPORTED = 6  /* the requested plan needs a path not built yet */
} toom_status;

/* Recursion plan (SURVEY.md §8 "reference shape"; SPEC.md:315-320 ToomPlan).
 * top_B: B of the top level: 3 (points 0,1,-1,2,inf), 4 (0,+-1,+-2,1/2,inf),
 *        8 (the paper's points 0,+-1,+-2,...,+-64) or
 *        16 (31 points: 0, inf and the 29 smallest-height +-p/q, homogeneous;
 *        BASELINE configs[4]) or 32 (the paper's points 0, +-2^j, j < 31: B = 32
 *        as the paper's 64-bit code allows; divisors up to 2^60
 *        run as exact divisions by their 32-bit word factors); 16 and 32 run
 *        on the limb-parallel long-vector kernels only;
 * lower levels: Toom-4 while the operand has more than t4 limbs, Toom-3
 *        while more than t3 limbs, schoolbook base case otherwise (<= 64 limbs);
 * chunk: products per scheduling chunk (0 = automatic);
 * long_count: which recursion levels run on the limb-parallel long-vector
 *        kernels (the upper levels of one large product: few, long
 *        operands); the levels below run one thread (or lane) per instance.
 *        0 = default: levels whose operands exceed 2048 limbs (environment
 *        overrides TOOM_LONG_MIN_N / TOOM_LONG_MAX_COUNT for tuning); 1 = never;
 *        k >= 2: levels with fewer than k instances.  Always a prefix of
 *        the recursion.                                                    */
typedef struct {
    int top_B;
    size_t t4;
    size_t t3;
    size_t chunk;
    size_t long_count;
} toom_plan_t;

/* Default plan for a given top B: t4 = 256, t3 = 64, chunk automatic. */
toom_plan_t toom_default_plan(int B);

/* w[i] = u[i] * v[i] for i < batch.
 * u, v: [batch][n] uint32 (row-major, device); w: [batch][2n] (device).
 * B: top-level B in {3, 4, 8, 16, 32} (see toom_plan_t).  n >= 1, batch >= 0
 * (batch 0: no-op).
 * Errors: TOOM_EINVAL (null/aliasing/B), TOOM_ENOMEM, TOOM_ECUDA.           */
toom_status toom_mul_batched(uint32_t *w, const uint32_t *u, const uint32_t *v,
                             size_t n, size_t batch, int B, void *stream);

/* As toom_mul_batched with an explicit plan (plan->top_B overrides B). */
toom_status toom_mul_batched_plan(uint32_t *w, const uint32_t *u, const uint32_t *v,
                                  size_t n, size_t batch, const toom_plan_t *plan,
                                  void *stream);

/* Squaring specialisation: w[i] = u[i]^2 for i < batch,
 * layouts as toom_mul_batched (u: [batch][n], w: [batch][2n], device).  The
 * evaluation runs once (V = U at every level, Eq. 1.1-1.2 for one operand) and
 * the base case squares: sum_{i<j} 2 a_i a_j + a_i^2, E(E+1)/2 instead of E^2
 * limb-products.  Errors as toom_mul_batched.  toom_mul with u == v and
 * nu == nv takes the same path.                                            */
toom_status toom_sqr_batched(uint32_t *w, const uint32_t *u, size_t n, size_t batch, const toom_plan_t *plan,
                             void *stream);

/* w[0 .. nu+nv) = u[0..nu) * v[0..nv) (device pointers).  nu, nv >= 0;
 * zero-length operands are zero (w is zeroed).  The shorter operand is
 * zero-padded to a common block width.                        */
toom_status toom_mul(uint32_t *w, const uint32_t *u, size_t nu, const uint32_t *v, size_t nv,
                     int B, void *stream);

/* Toom as a top-level wrapper over a different inner multiplier (PAPER.md
 * §5, :188-196: Toom-Cook "as a top-level threading wrapper" around GMP's FFT;
 * SURVEY.md §8(f)4).  w[0 .. nu+nv) = u * v (device pointers, nu, nv >= 1):
 * B in {3, 4, 8, 16, 32}: the Toom-B top level on the long-vector kernels
 * (evaluation at the 2B-1 points, interpolation, recomposition), its 2B-1
 * pointwise products by an exact number-theoretic transform over the prime
 * p = 2^64 - 2^32 + 1 (16-bit digits; every convolution coefficient < 2^53 < p);
 * B = 0: the NTT product alone.  Errors as toom_mul.                        */
toom_status toom_mul_ntt(uint32_t *w, const uint32_t *u, size_t nu, const uint32_t *v, size_t nv, int B,
                         void *stream);

/* End-to-end variant with HOST buffers (pinned or pageable): copies u, v to
 * the device, multiplies, copies w back, and synchronizes `stream` before
 * returning.  Layouts as toom_mul_batched.                                 */
toom_status toom_mul_batched_host(uint32_t *w_host, const uint32_t *u_host, const uint32_t *v_host,
                                  size_t n, size_t batch, const toom_plan_t *plan, void *stream);

/* Device workspace (bytes) that toom_mul_batched_plan needs for this shape:
 * the breadth-first recursion keeps every level's child operands and products
 * (2B-1 per parent, Eq. 2.1) plus the long levels' scan state
 * (SURVEY.md §5(g), H5).  0 on an invalid plan.  Covers every plan, including
 * the schoolbook-only one (n <= 64).                                       */
size_t toom_workspace_bytes(size_t n, size_t batch, const toom_plan_t *plan);

/* Provide a caller-owned device workspace (NULL, 0 = let the library
 * allocate and cache its own).  Ownership stays with the caller; the library
 * uses it until replaced and never frees it.  Without one, the library keeps
 * one buffer PER STREAM (calls on different streams never share scratch).
 * A caller buffer is shared by all streams: a call on another stream than the
 * previous user's waits (stream-ordered) for that user's work first.  A call
 * whose shape needs more than `bytes` fails with TOOM_ENOMEM.  Blocks until
 * work using the previous buffers has finished.                            */
toom_status toom_set_workspace(void *dev_ptr, size_t bytes);

/* Status of the last failed call on this host thread (TOOM_OK if none);
 * reading it clears it.  When toom_set_check / toom_set_verify are on, it
 * first synchronizes the device and reports a device-detected failure of any
 * call since the last read: TOOM_EINEXACT (an "exact" division left a
 * remainder, §3; SPEC.md:462 exit code 3) or TOOM_EVERIFY (the
 * result's residue mod 2^61-1 differs from the residues' product).         */
toom_status toom_last_error(void);

/* Debug exact-division check: every
 * interpolation kernel of the batched path whose dividends have a known end
 * (fused bottom rows, top-level rows, row-parallel levels) checks that the
 * 2-adic division left no remainder (final borrow) and that the power-of-two
 * shift dropped only zero bits.  on = 0 (default): no checks.             */
void toom_set_check(int on);

/* Result verification: after every unsigned product (toom_mul,
 * toom_mul_batched*), a kernel checks w mod p == (u mod p)(v mod p) mod p
 * for p = 2^61 - 1 (one warp per product, O(n) reads).  Catches any wrong
 * limb of w with probability 1 - 2^-61 per random error.  on = 0: off.   */
void toom_set_verify(int on);

/* Fault injection for tests: kind 1 flips one bit of one
 * base-case product inside the fused bottom kernel, so that the next exact
 * division is inexact; kind 2 injects no fault but sends every product of
 * the C2 top level (csrc/toplevel_cls.cuh) through the serial carry/borrow
 * chain that otherwise runs only when a carry wraps a segment's limb 0;
 * 0 = off.  Never set in production.                                      */
void toom_debug_fault(int kind);

/* Human-readable name of a status code (static string). */
const char *toom_status_string(toom_status s);

/* Number of kernels the last compute call launched (instrumentation for
 * bench.py's "gpu_launches"). */
size_t toom_last_launch_count(void);

/* ---- instrumentation (bench.py) ---------------------------------------- */

/* When enabled, every kernel the library launches on this host thread is
 * bracketed by CUDA events on its stream (adds a little overhead; bench.py
 * uses it in a separate pass after the timed region). */
void toom_profile_enable(int on);

/* Synchronizes the device and sums, per kernel category (0 evaluation,
 * 1 base case, 2 interpolation+recomposition, 3 other), the event-timed
 * milliseconds and launch counts recorded since the last collect.  Writes
 * ncat entries; returns the number of categories the library knows. */
int toom_profile_collect(double *ms, size_t *launches, int ncat);

/* JSON description of the recursion plan for this shape (levels: B, count,
 * n, b, e, Lw, npts; workspace bytes).  Writes at most len bytes to buf
 * (NUL-terminated); returns the length needed including the NUL, 0 on error. */
size_t toom_plan_describe(size_t n, size_t batch, const toom_plan_t *plan, char *buf, size_t len);

/* Microbenchmark of the limb-product peak: the issue rate of the 32x32->64
 * integer MAD (mad.wide.u32 -> IMAD.WIDE.U32; one limb-product each), 148 SMs
 * x 8 CTAs x 256 threads x 8 independent chains.  Used as the "alu" roofline
 * peak.  Runs on `stream`, synchronizes, returns limb-products per second
 * (and the elapsed ms in *ms), or a negative value on error. */
double toom_probe_limb_products(double *ms, void *stream);

/* As above for the schoolbook kernel's own per-limb-product sequence
 * (mad.lo.cc / madc.hi.cc / addc carry-flag chains), for context. */
double toom_probe_carry_chain(double *ms, void *stream);

/* Enable (default) or disable the fused bottom-level kernel (evaluation,
 * base-case products, interpolation and recomposition of the last Toom level
 * in one kernel, in shared memory).  Disabled, that level runs as separate
 * staged launches through HBM; results are identical (tests compare both). */
void toom_set_fused(int on);

/* Top-level interpolation of batched Toom-3/Toom-4 products: 3 = one warp
 * per product over the common-denominator matrix form with a warp
 * carry/borrow scan (k_interp_top_warp; used when the fused level is directly
 * below, else mode 2); 2 (default) = products of a group of instances staged
 * in shared memory, rows in place, then recomposition (k_interp_top_smem); 1 = one
 * streaming pass per product (k_interp_top_stream); 0 = the per-row kernel
 * (k_interp_top_rows) and, for every batched level, the one-thread-per-
 * product streaming programs; 4 = row-parallel interpolation (one thread per
 * coefficient row and product) + segment-parallel recomposition at every
 * batched Toom-3/4 level.  The paper's Toom-8 top level (C3) uses the
 * row-parallel form unless the mode is 0.  All are exact; tests compare them. */
void toom_set_top_stream(int on);

/* Toom-16 top-level interpolation: 1 (default) = the matrix form (even-odd
 * split, then one dense pass per half with the symbolic inverse's wide
 * multipliers and exact divisions by the rows' word-factored denominators,
 * PAPER.md:162); 0 = the staged Newton program (the
 * paper's listings, one long op per step).  Both
 * are exact; tests compare them.  Affects later calls only.                */
void toom_set_t16_matrix(int on);

/* C2-shaped batches (256-limb operands, Toom-4 -> Toom-4 -> 18-limb
 * schoolbook, reading 18).  mode 2 (default): the bottom level
 * forms X = 360 y in the common-denominator matrix form (no
 * division) and the top level runs ONE exact division by 360^2 over its own
 * common-denominator sum, split into segments by the closed-form 2-adic
 * borrow; 1: the bottom divides its rows itself, the top divides by 360 the
 * same way; 0: both levels divide row by row (the listing rows, PAPER.md:
 * 114-120, 154-158, composed).  Same results; tests compare all three.
 * Affects later calls only.                                              */
void toom_set_c2_mode(int mode);

/* Single large products (C4, C5): 1 (default) = the Toom-3 bottom level
 * right under the lazy Toom-4 levels forms X = 6 y without dividing
 * (PAPER.md:162 matrix form) and the factor 6 joins the lazy block's
 * finishing division (readings 18, 19); 0 = the bottom divides
 * its rows itself.  Same results; tests compare both.  Affects later calls. */
void toom_set_lazy_bottom(int on);

/* ---- stage exports (tests, bench) ------------------------------------- */

/* Base case alone (step a3): batched schoolbook of signed two's-complement
 * operands.  u, v: INTERLEAVED [E][count] (limb-major: limb i of instance c
 * at i*count + c), w: [2E][count] interleaved; 1 <= E <= 64.               */
toom_status toom_base_interleaved(uint32_t *w, const uint32_t *u, const uint32_t *v,
                                  size_t E, size_t count, void *stream);

/* The same base case on the 5th-generation tensor cores (SURVEY.md §8(f)2,
 * an experiment: north_star allows tensor cores only where they beat the
 * integer-MAD path; the paper is silent on the base case):
 * |u|, |v| as 4E bytes, one tcgen05.mma.cta_group::1.kind::i8 per product
 * (M = 128 rows of the Toeplitz byte windows of |u|, N = 16 >= ceil(4E/32)
 * reversed 32-byte chunks of |v|, K = 32, u8 x u8 -> s32 in TMEM, exact:
 * every partial sum < 2^21), byte columns summed and carried into 2E limbs,
 * the sign applied.  Same layout and result as toom_base_interleaved.
 * E in {2, 5, 9, 16, 17, 18, 23, 24} (compiled instances), else
 * TOOM_EUNSUPPORTED.  Not used by the multiplication paths.              */
toom_status toom_base_interleaved_tc(uint32_t *w, const uint32_t *u, const uint32_t *v,
                                     size_t E, size_t count, void *stream);

/* Evaluation alone (step a2) at the top level: for each of the `batch`
 * unsigned operands a[batch][n], the 2B-1 values at the point set of B,
 * written INTERLEAVED as out[e][npoints*batch] (value of point k of operand
 * i at column k*batch + i), two's complement, e = toom_eval_width(n, B).    */
toom_status toom_eval_top(uint32_t *out, const uint32_t *a, size_t n, size_t batch, int B, void *stream);
size_t toom_eval_width(size_t n, int B);
int toom_npoints(int B);

/* ---- long-path stage exports (sharded top level, C5; SURVEY.md §8(b),(e)) --
 * These run one top Toom level of `batch` instances on the limb-parallel
 * long-vector kernels, so that the 2B-1 top-level products can be computed
 * on other GPUs (Eq. 2.5).  B in {3, 4, 8, 16};
 * e = toom_eval_width(n, B); all values two's complement little-endian.     */

/* Step a1+a2: out[k][i][0..e) = A_i(x_k) for every point k of B's point set
 * (homogeneous evaluation sum_j a_ij p^j q^(B-1-j), Eq. 1.1-1.2), where
 * a[i][0..n) is split into B blocks of ceil(n/B) limbs.  a is unsigned
 * (is_signed = 0) or two's complement (is_signed = 1).  out: device,
 * [2B-1][batch][e], must not overlap a.                                     */
toom_status toom_eval_points(uint32_t *out, const uint32_t *a, size_t n, size_t batch, int B,
                             int is_signed, void *stream);

/* As toom_eval_points for the points k0 <= k < k1 only (0 <= k0 <= k1 <=
 * 2B-1): out[k - k0][i][0..e).  Each rank of the sharded top level (Eq. 2.5,
 * PAPER.md:44-46) evaluates its own points from broadcast operands.  An
 * empty range (k0 == k1) is a no-op and out may be null.
 * Errors: TOOM_EINVAL (range, pointers, overlap), TOOM_ECUDA.               */
toom_status toom_eval_points_range(uint32_t *out, const uint32_t *a, size_t n, size_t batch, int B,
                                   int is_signed, int k0, int k1, void *stream);

/* Steps a4+a5: from the 2B-1 pointwise products y[k][i][0..2e) (Eq. 2.1,
 * two's complement), interpolate the coefficients w_0..w_{2B-2} (even-odd
 * method, Eqs. 4.5-4.6, with the listings PAPER.md:114-120, 154-158 or their
 * matrix form PAPER.md:162; exact divisions) and recompose
 * w[i][0..2n) = sum_j w_j 2^(32 b j) (Eq. 1.3).  w must not overlap y.      */
toom_status toom_interp_recompose(uint32_t *w, const uint32_t *y, size_t n, size_t batch, int B,
                                  void *stream);

/* As toom_mul_batched_plan for two's-complement operands u[i], v[i] of n
 * limbs; w[i] gets the 2n-limb two's-complement product.  The top level must
 * be a long-vector level (batch < plan->long_count or its default), else
 * TOOM_EUNSUPPORTED.  Used for the sharded top-level products of C5.       */
toom_status toom_mul_signed_batched(uint32_t *w, const uint32_t *u, const uint32_t *v, size_t n,
                                    size_t batch, const toom_plan_t *plan, void *stream);

/* 2e: limbs of one pointwise product of toom_eval_points' outputs. */
size_t toom_product_width_point(size_t n, int B);

#ifdef __cplusplus
}
#endif
#endif /* TOOMGPU_H */
