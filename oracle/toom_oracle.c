/*
 * oracle/toom_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * The plain, slow, obviously-correct CPU oracle for the B-way Toom-Cook
 * multiplication of Kronenburg, "Toom-Cook Multiplication: Some Theoretical
 * and Practical Aspects" (arXiv 1602.02740; /root/reference/PAPER.md).
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library.  The product (the CUDA path
 * under paper_1602_02740_b200/) never links, imports or calls it, and this
 * file shares no code, header, table or constant generator with it.
 *
 * Contents (each function cites the passage it follows):
 *   O1  oracle_schoolbook        -- the definition w = u*v, digit by digit
 *   O2  oracle_toom              -- recursive Toom-Cook written step by step in
 *                                   the paper's order: split (Eq. 1.1), evaluate
 *                                   at 0 and +-2^j (Eq. 4.1),
 *                                   2B-1 recursive products (Eq. 2.1),
 *                                   even-odd split (Eqs. 4.5-4.6),
 *                                   divided differences (listing PAPER.md:114-120),
 *                                   Newton -> monomial (listing PAPER.md:154-158),
 *                                   recomposition w = W(2^b) (Eq. 1.3)
 *   O3  oracle_mod / oracle_is_prime_u64 -- residues w mod p (ring homomorphism)
 *   listings exposed for pins: oracle_interp_listings, oracle_even_odd_interp
 *
 * Arithmetic: sign-magnitude big integers on uint32 limbs (the paper's 32-bit
 * words).  Exact divisions are done by plain top-down long
 * division with the remainder checked (SPEC.md:89-97 design decision); a
 * nonzero remainder sets the sticky `inexact` flag (PAPER.md:122 says every
 * such division is exact, so a nonzero remainder is a bug).
 *
 * Parity pins: see tests/test_oracle_pins.py (every function above is pinned;
 * nothing here is "parity unpinned").
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>
#include <pthread.h>

typedef uint32_t limb_t;

/* ------------------------------------------------------------------------- */
/* sign-magnitude big integer                                                 */
/* ------------------------------------------------------------------------- */
typedef struct {
    limb_t *d;   /* little-endian magnitude, normalized: n==0 or d[n-1]!=0 */
    size_t n;
    int neg;     /* 1 if negative; zero is always non-negative */
} bigint;

static _Thread_local int g_inexact = 0;      /* sticky: a "exact" division left a remainder */
static _Thread_local int g_skip_division = -1; /* fault injection: skip the k-th listing-1 division */
static _Thread_local long g_division_counter = 0;
static _Thread_local long g_products[64];    /* products computed per recursion depth (Eq. 2.1) */
static _Thread_local int g_top_threads = 1;  /* P processors on the top-level products (Eq. 2.5) */

static void *xmalloc(size_t bytes) {
    void *p = malloc(bytes ? bytes : 1);
    if (!p) abort();
    return p;
}

static bigint bi_new(size_t cap) {
    bigint r;
    r.d = (limb_t *)xmalloc(sizeof(limb_t) * (cap ? cap : 1));
    r.n = 0;
    r.neg = 0;
    return r;
}

static void bi_free(bigint *a) {
    free(a->d);
    a->d = NULL;
    a->n = 0;
    a->neg = 0;
}

static void bi_norm(bigint *a) {
    while (a->n && a->d[a->n - 1] == 0) a->n--;
    if (a->n == 0) a->neg = 0;
}

static bigint bi_from_limbs(const limb_t *p, size_t n) {
    bigint r = bi_new(n);
    if (n) memcpy(r.d, p, n * sizeof(limb_t));
    r.n = n;
    bi_norm(&r);
    return r;
}

static bigint bi_copy(const bigint *a) {
    bigint r = bi_from_limbs(a->d, a->n);
    r.neg = a->neg;
    return r;
}

/* compare magnitudes */
static int mag_cmp(const limb_t *a, size_t an, const limb_t *b, size_t bn) {
    if (an != bn) return an < bn ? -1 : 1;
    for (size_t i = an; i-- > 0;) {
        if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    }
    return 0;
}

/* |a| + |b| */
static bigint mag_add(const bigint *a, const bigint *b) {
    size_t n = a->n > b->n ? a->n : b->n;
    bigint r = bi_new(n + 1);
    uint64_t carry = 0;
    for (size_t i = 0; i < n; i++) {
        uint64_t s = carry;
        if (i < a->n) s += a->d[i];
        if (i < b->n) s += b->d[i];
        r.d[i] = (limb_t)s;
        carry = s >> 32;
    }
    r.d[n] = (limb_t)carry;
    r.n = n + 1;
    bi_norm(&r);
    return r;
}

/* |a| - |b|, requires |a| >= |b| */
static bigint mag_sub(const bigint *a, const bigint *b) {
    bigint r = bi_new(a->n);
    uint64_t borrow = 0;
    for (size_t i = 0; i < a->n; i++) {
        uint64_t bi = (i < b->n ? b->d[i] : 0) + borrow;
        uint64_t ai = a->d[i];
        if (ai >= bi) {
            r.d[i] = (limb_t)(ai - bi);
            borrow = 0;
        } else {
            r.d[i] = (limb_t)(ai + ((uint64_t)1 << 32) - bi);
            borrow = 1;
        }
    }
    r.n = a->n;
    bi_norm(&r);
    return r;
}

/* a + b, signed (SPEC.md:98-106 int_arith) */
static bigint bi_add(const bigint *a, const bigint *b) {
    bigint r;
    if (a->neg == b->neg) {
        r = mag_add(a, b);
        r.neg = a->neg;
    } else if (mag_cmp(a->d, a->n, b->d, b->n) >= 0) {
        r = mag_sub(a, b);
        r.neg = a->neg;
    } else {
        r = mag_sub(b, a);
        r.neg = b->neg;
    }
    bi_norm(&r);
    return r;
}

/* a - b, signed */
static bigint bi_sub(const bigint *a, const bigint *b) {
    bigint nb = *b; /* shallow: flip sign only */
    nb.neg = b->n ? !b->neg : 0;
    return bi_add(a, &nb);
}

/* a * 2^s  ("many multiplications reduce to shifts") */
static bigint bi_shl(const bigint *a, unsigned s) {
    size_t q = s / 32;
    unsigned r = s % 32;
    bigint out = bi_new(a->n + q + 1);
    memset(out.d, 0, sizeof(limb_t) * (a->n + q + 1));
    for (size_t i = 0; i < a->n; i++) {
        uint64_t x = (uint64_t)a->d[i] << r;
        out.d[i + q] |= (limb_t)x;
        out.d[i + q + 1] |= (limb_t)(x >> 32);
    }
    out.n = a->n + q + 1;
    out.neg = a->neg;
    bi_norm(&out);
    return out;
}

/* a * m for one word m */
static bigint bi_mul_word(const bigint *a, limb_t m) {
    bigint r = bi_new(a->n + 1);
    uint64_t carry = 0;
    for (size_t i = 0; i < a->n; i++) {
        uint64_t t = (uint64_t)a->d[i] * m + carry;
        r.d[i] = (limb_t)t;
        carry = t >> 32;
    }
    r.d[a->n] = (limb_t)carry;
    r.n = a->n + 1;
    r.neg = a->neg;
    bi_norm(&r);
    return r;
}

/* a / d for one word d, exact: top-down long division with a running
 * remainder; a nonzero remainder means the division was not exact, which
 * PAPER.md:122 ("the divisions are exact integer divisions [4]") rules out,
 * so it is recorded in g_inexact. */
static bigint bi_divexact_word(const bigint *a, limb_t d) {
    bigint q = bi_new(a->n);
    uint64_t rem = 0;
    for (size_t i = a->n; i-- > 0;) {
        uint64_t cur = (rem << 32) | a->d[i];
        q.d[i] = (limb_t)(cur / d);
        rem = cur % d;
    }
    q.n = a->n;
    q.neg = a->neg;
    if (rem != 0) g_inexact = 1;
    bi_norm(&q);
    return q;
}

/* ------------------------------------------------------------------------- */
/* O1: schoolbook -- the definition of w = u*v.                                */
/* w[0 .. nu+nv) = u[0..nu) * v[0..nv), uint32 limbs, little-endian.          */
/* ------------------------------------------------------------------------- */
void oracle_schoolbook(const limb_t *u, size_t nu, const limb_t *v, size_t nv, limb_t *w) {
    for (size_t k = 0; k < nu + nv; k++) w[k] = 0;
    for (size_t i = 0; i < nu; i++) {
        uint64_t carry = 0;
        for (size_t j = 0; j < nv; j++) {
            uint64_t t = (uint64_t)u[i] * v[j] + w[i + j] + carry;
            w[i + j] = (limb_t)t;
            carry = t >> 32;
        }
        w[i + nv] = (limb_t)carry;
    }
}

static bigint bi_mul_schoolbook(const bigint *a, const bigint *b) {
    bigint r = bi_new(a->n + b->n);
    oracle_schoolbook(a->d, a->n, b->d, b->n, r.d);
    r.n = a->n + b->n;
    r.neg = a->neg ^ b->neg;
    bi_norm(&r);
    return r;
}

/* ------------------------------------------------------------------------- */
/* §3 listings on arrays of big integers                                      */
/* ------------------------------------------------------------------------- */

/* PAPER.md:114-120 (§3, Theorem 3.2, Eq. 3.8):
 *   for(k=0;k<=n;k++) coeff[k] = y[k];
 *   for(k=1;k<=n;k++)
 *     for(m=n;m>=k;m--)
 *       coeff[m] = (coeff[m]-coeff[m-1])/(x[m]-x[m-k]);
 * The abscissas are non-negative and increasing here, so x[m]-x[m-k] > 0. */
static void listing_divided_differences(int n, const int64_t *x, bigint *coeff) {
    for (int k = 1; k <= n; k++) {
        for (int m = n; m >= k; m--) {
            bigint diff = bi_sub(&coeff[m], &coeff[m - 1]);
            int64_t den = x[m] - x[m - k];
            bigint q;
            int neg_den = den < 0;
            uint64_t aden = neg_den ? (uint64_t)(-den) : (uint64_t)den;
            if (g_skip_division >= 0 && g_division_counter++ == g_skip_division) {
                q = bi_copy(&diff); /* fault injection: the division is skipped */
                g_inexact = 1;      /* ... which the residue/exactness checks must catch */
            } else {
                q = bi_divexact_word(&diff, (limb_t)aden);
                if (neg_den && q.n) q.neg = !q.neg;
            }
            bi_free(&diff);
            bi_free(&coeff[m]);
            coeff[m] = q;
        }
    }
}

/* PAPER.md:154-158 (§3, Theorem 3.3, Eq. 3.17):
 *   for(m=n-1;m>=0;m--)
 *     for(k=m;k<=n-1;k++)
 *       coeff[k] -= x[m] * coeff[k+1];                                      */
static void listing_newton_to_monomial(int n, const int64_t *x, bigint *coeff) {
    for (int m = n - 1; m >= 0; m--) {
        for (int k = m; k <= n - 1; k++) {
            int64_t xm = x[m];
            uint64_t axm = xm < 0 ? (uint64_t)(-xm) : (uint64_t)xm;
            bigint t = bi_mul_word(&coeff[k + 1], (limb_t)axm);
            if (xm < 0 && t.n) t.neg = !t.neg;
            bigint r = bi_sub(&coeff[k], &t);
            bi_free(&t);
            bi_free(&coeff[k]);
            coeff[k] = r;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* O2: recursive Toom-Cook, the paper's method step by step                   */
/* ------------------------------------------------------------------------- */
typedef struct {
    int top_B;       /* B at depth 0 (2..16); 0 = use the size rule below */
    size_t t4;       /* Toom-4 while n > t4 (depth >= 1) */
    size_t t3;       /* Toom-3 while n > t3; schoolbook at n <= t3 */
} oracle_plan;

static int plan_B(const oracle_plan *p, int depth, size_t n) {
    if (depth == 0 && p->top_B >= 2) return p->top_B;
    if (n > p->t4) return 4;
    if (n > p->t3) return 3;
    return 0; /* schoolbook */
}

static bigint toom_rec(const bigint *u, const bigint *v, const oracle_plan *plan, int depth);

/* y = a*b for signed a, b: magnitudes multiplied recursively (Eq. 2.1),
 * sign = sign(a) xor sign(b). */
static bigint signed_product(const bigint *a, const bigint *b, const oracle_plan *plan, int depth) {
    bigint am = *a, bm = *b;
    am.neg = 0;
    bm.neg = 0;
    bigint y = toom_rec(&am, &bm, plan, depth);
    y.neg = (a->neg ^ b->neg) && y.n;
    return y;
}

/* one pointwise product y = a*b of the Toom level (Eq. 2.1) */
typedef struct {
    bigint a, b, y;
    const oracle_plan *plan;
    int depth;
    int inexact;
    long products[64];
} prod_task;

typedef struct {
    prod_task *tasks;
    int ntask, tid, nthr;
} prod_worker;

static void *prod_worker_main(void *arg) {
    prod_worker *w = (prod_worker *)arg;
    for (int t = w->tid; t < w->ntask; t += w->nthr) {
        prod_task *k = &w->tasks[t];
        g_inexact = 0;
        memset(g_products, 0, sizeof g_products);
        k->y = signed_product(&k->a, &k->b, k->plan, k->depth);
        k->inexact = g_inexact;
        memcpy(k->products, g_products, sizeof g_products);
        bi_free(&k->a);
        bi_free(&k->b);
    }
    return NULL;
}

/* the products of one level, on `nthr` threads (independent: Eq. 2.5); the
 * workers' sticky inexact flags and per-depth counters are merged back */
static void run_products(prod_task *tasks, int ntask, int nthr) {
    if (nthr > ntask) nthr = ntask;
    if (nthr <= 1) {
        for (int t = 0; t < ntask; t++) {
            tasks[t].y = signed_product(&tasks[t].a, &tasks[t].b, tasks[t].plan, tasks[t].depth);
            bi_free(&tasks[t].a);
            bi_free(&tasks[t].b);
        }
        return;
    }
    pthread_t *th = (pthread_t *)xmalloc(sizeof(pthread_t) * nthr);
    prod_worker *ws = (prod_worker *)xmalloc(sizeof(prod_worker) * nthr);
    for (int i = 0; i < nthr; i++) {
        ws[i].tasks = tasks; ws[i].ntask = ntask; ws[i].tid = i; ws[i].nthr = nthr;
        pthread_create(&th[i], NULL, prod_worker_main, &ws[i]);
    }
    for (int i = 0; i < nthr; i++) pthread_join(th[i], NULL);
    for (int t = 0; t < ntask; t++) {
        g_inexact |= tasks[t].inexact;
        for (int d = 0; d < 64; d++) g_products[d] += tasks[t].products[d];
    }
    free(th);
    free(ws);
}

/* Split |a| into B blocks of b limbs (Eq. 1.1: u = U(2^b)); blocks past the
 * end are zero (the shorter operand is zero-padded). */
static void split_blocks(const bigint *a, int B, size_t b, bigint *blk) {
    for (int k = 0; k < B; k++) {
        size_t lo = (size_t)k * b;
        size_t len = 0;
        if (lo < a->n) len = (a->n - lo) < b ? (a->n - lo) : b;
        blk[k] = bi_from_limbs(a->d + (lo < a->n ? lo : 0), len);
    }
}

/* E = sum_{k even} u_k 2^{jk},  O = sum_{k odd} u_k 2^{jk}  (Eq. 4.1 with
 * x = 2^j; "many multiplications reduce to shifts").
 * U(2^j) = E + O, U(-2^j) = E - O (Eqs. 4.3-4.4).                          */
static void eval_pair(const bigint *blk, int B, unsigned j, bigint *plus, bigint *minus) {
    bigint E = bi_new(1), O = bi_new(1);
    for (int k = 0; k < B; k++) {
        bigint t = bi_shl(&blk[k], j * (unsigned)k);
        bigint *acc = (k % 2 == 0) ? &E : &O;
        bigint s = bi_add(acc, &t);
        bi_free(acc);
        *acc = s;
        bi_free(&t);
    }
    *plus = bi_add(&E, &O);
    *minus = bi_sub(&E, &O);
    bi_free(&E);
    bi_free(&O);
}

static bigint toom_rec(const bigint *u, const bigint *v, const oracle_plan *plan, int depth) {
    size_t nmax = u->n > v->n ? u->n : v->n;
    size_t nmin = u->n < v->n ? u->n : v->n;
    if (depth < 64) g_products[depth]++;
    if (nmin == 0) return bi_new(1);
    int B = plan_B(plan, depth, nmax);
    if (B < 2 || nmax < (size_t)B) return bi_mul_schoolbook(u, v);

    int n = B - 1;                              /* degree, B = n+1 */
    size_t b = (nmax + (size_t)B - 1) / (size_t)B;  /* block width in limbs */

    bigint *ub = (bigint *)xmalloc(sizeof(bigint) * B);
    bigint *vb = (bigint *)xmalloc(sizeof(bigint) * B);
    split_blocks(u, B, b, ub);
    split_blocks(v, B, b, vb);

    /* points: x_0 = 0 and +-2^j, j = 0..n-1 (PAPER.md:200 + §4): 2n+1 = 2B-1 products.
     * Evaluate every point first (Eq. 4.1, 4.3-4.4), then form the products
     * (Eq. 2.1) -- at depth 0 on P threads (Eq. 2.5). */
    prod_task *tasks = (prod_task *)xmalloc(sizeof(prod_task) * (2 * n + 1));
    tasks[0].a = bi_copy(&ub[0]);                 /* U(0) = u_0 */
    tasks[0].b = bi_copy(&vb[0]);
    for (int j = 0; j < n; j++) {
        eval_pair(ub, B, (unsigned)j, &tasks[1 + 2 * j].a, &tasks[2 + 2 * j].a);
        eval_pair(vb, B, (unsigned)j, &tasks[1 + 2 * j].b, &tasks[2 + 2 * j].b);
    }
    for (int t = 0; t < 2 * n + 1; t++) { tasks[t].plan = plan; tasks[t].depth = depth + 1; }
    run_products(tasks, 2 * n + 1, depth == 0 ? g_top_threads : 1);
    bigint W0 = tasks[0].y;                       /* W(0) = U(0)V(0) */
    bigint *We = (bigint *)xmalloc(sizeof(bigint) * (n + 1));
    bigint *Wo = (bigint *)xmalloc(sizeof(bigint) * (n + 1));
    int64_t *z = (int64_t *)xmalloc(sizeof(int64_t) * (n + 1));
    z[0] = 0;
    We[0] = bi_copy(&W0);          /* even problem: first point (0, W(0)) */
    Wo[0] = bi_new(1);             /* odd problem: first point (0, 0) */
    for (int j = 0; j < n; j++) {
        bigint yp = tasks[1 + 2 * j].y;    /* W(x)  */
        bigint ym = tasks[2 + 2 * j].y;    /* W(-x) */
        /* Eq. 4.5: W_e(x^2) = (W(x) + W(-x)) / 2 */
        bigint s = bi_add(&yp, &ym);
        We[j + 1] = bi_divexact_word(&s, 2);
        /* Eq. 4.6 times x^2: x^2 W_o(x^2) = x (W(x) - W(-x)) / 2 */
        bigint d = bi_sub(&yp, &ym);
        bigint dx = bi_shl(&d, (unsigned)j);
        Wo[j + 1] = bi_divexact_word(&dx, 2);
        z[j + 1] = (int64_t)1 << (2 * j);   /* z = x^2 = 4^j <= 2^28 for B = 16 */
        bi_free(&s); bi_free(&d); bi_free(&dx);
        bi_free(&yp); bi_free(&ym);
    }
    free(tasks);

    /* the two degree-n interpolations (independent) */
    listing_divided_differences(n, z, We);
    listing_newton_to_monomial(n, z, We);
    listing_divided_differences(n, z, Wo);
    listing_newton_to_monomial(n, z, Wo);
    if (Wo[0].n != 0) g_inexact = 1;   /* x^2 W_o has no constant term */

    /* interleave ("the resulting coefficients move one place
     * higher"): w_{2k} = We[k], w_{2k+1} = Wo[k+1]; then w = W(2^b) (Eq. 1.3) */
    bigint acc = bi_new(1);
    for (int k = 2 * n; k >= 0; k--) {
        bigint shifted = bi_shl(&acc, (unsigned)(32 * b));   /* Horner in 2^b */
        const bigint *wk = (k % 2 == 0) ? &We[k / 2] : &Wo[(k - 1) / 2 + 1];
        bigint s = bi_add(&shifted, wk);
        bi_free(&shifted);
        bi_free(&acc);
        acc = s;
    }
    if (acc.neg) g_inexact = 1;   /* a product of magnitudes is never negative */

    for (int k = 0; k < B; k++) { bi_free(&ub[k]); bi_free(&vb[k]); }
    for (int k = 0; k <= n; k++) { bi_free(&We[k]); bi_free(&Wo[k]); }
    free(ub); free(vb); free(We); free(Wo); free(z);
    bi_free(&W0);
    return acc;
}

/* ------------------------------------------------------------------------- */
/* exported API (ctypes)                                                      */
/* ------------------------------------------------------------------------- */

/* w[0 .. nu+nv) = u * v by recursive Toom-Cook with the paper's points.
 * top_B: B of the top level (2..16), 0 = size rule; t4, t3: thresholds of
 * the lower levels (Toom-4 while n > t4, Toom-3 while n > t3, else schoolbook).
 * Returns 0, or 3 if any "exact" division left a remainder (SPEC.md:462 exit
 * code 3). */
int oracle_toom(const limb_t *u, size_t nu, const limb_t *v, size_t nv, limb_t *w,
                int top_B, size_t t4, size_t t3) {
    g_top_threads = 1;
    oracle_plan plan = {top_B, t4, t3};
    int saved = g_inexact;
    g_inexact = 0;
    bigint a = bi_from_limbs(u, nu), b = bi_from_limbs(v, nv);
    bigint r = toom_rec(&a, &b, &plan, 0);
    for (size_t i = 0; i < nu + nv; i++) w[i] = i < r.n ? r.d[i] : 0;
    int bad = g_inexact || r.n > nu + nv;
    bi_free(&a); bi_free(&b); bi_free(&r);
    g_inexact = saved || bad;
    return bad ? 3 : 0;
}

/* as oracle_toom with the top-level products on `threads` host threads
 * (Eq. 2.5: P processors on the 2B-1 top-level products) */
int oracle_toom_mt(const limb_t *u, size_t nu, const limb_t *v, size_t nv, limb_t *w,
                   int top_B, size_t t4, size_t t3, int threads) {
    oracle_plan plan = {top_B, t4, t3};
    int saved = g_inexact;
    g_inexact = 0;
    g_top_threads = threads > 1 ? threads : 1;
    bigint a = bi_from_limbs(u, nu), b = bi_from_limbs(v, nv);
    bigint r = toom_rec(&a, &b, &plan, 0);
    g_top_threads = 1;
    for (size_t i = 0; i < nu + nv; i++) w[i] = i < r.n ? r.d[i] : 0;
    int bad = g_inexact || r.n > nu + nv;
    bi_free(&a); bi_free(&b); bi_free(&r);
    g_inexact = saved || bad;
    return bad ? 3 : 0;
}

/* batched: u, v are [batch][n], w is [batch][2n] */
int oracle_toom_batched(const limb_t *u, const limb_t *v, limb_t *w, size_t n, size_t batch,
                        int top_B, size_t t4, size_t t3) {
    int st = 0;
    for (size_t i = 0; i < batch; i++) {
        int s = oracle_toom(u + i * n, n, v + i * n, n, w + i * 2 * n, top_B, t4, t3);
        if (s) st = s;
    }
    return st;
}

void oracle_schoolbook_batched(const limb_t *u, const limb_t *v, limb_t *w, size_t n, size_t batch) {
    for (size_t i = 0; i < batch; i++) oracle_schoolbook(u + i * n, n, v + i * n, n, w + i * 2 * n);
}

/* instrumentation for the "M = 2B-1 products" pin (Eq. 2.1) */
void oracle_reset_counters(void) {
    memset(g_products, 0, sizeof(g_products));
    g_division_counter = 0;
}
long oracle_products_at_depth(int depth) { return (depth >= 0 && depth < 64) ? g_products[depth] : -1; }
void oracle_set_fault_skip_division(int k) { g_skip_division = k; g_division_counter = 0; }

/* ---- listings on caller arrays, for the pins ----------------------------- */
/* values are fixed-width two's complement, `width` limbs each */
static bigint bi_from_twos(const limb_t *p, size_t width) {
    int neg = width && (p[width - 1] >> 31);
    bigint r = bi_new(width);
    if (!neg) {
        memcpy(r.d, p, width * sizeof(limb_t));
    } else {
        uint64_t carry = 1;
        for (size_t i = 0; i < width; i++) {
            uint64_t t = (uint64_t)(limb_t)~p[i] + carry;
            r.d[i] = (limb_t)t;
            carry = t >> 32;
        }
    }
    r.n = width;
    r.neg = neg;
    bi_norm(&r);
    return r;
}

static int bi_to_twos(const bigint *a, limb_t *p, size_t width) {
    if (a->n > width) return 1;
    for (size_t i = 0; i < width; i++) p[i] = i < a->n ? a->d[i] : 0;
    if (a->neg) {
        uint64_t carry = 1;
        for (size_t i = 0; i < width; i++) {
            uint64_t t = (uint64_t)(limb_t)~p[i] + carry;
            p[i] = (limb_t)t;
            carry = t >> 32;
        }
    }
    /* overflow if the sign bit disagrees */
    if (width && a->n && ((p[width - 1] >> 31) != (limb_t)a->neg)) return 1;
    return 0;
}

/* Runs listing 1 (divided differences) then listing 2 (Newton -> monomial)
 * on n+1 points x[0..n], values y (two's complement, `width` limbs each).
 * alpha_out receives the alpha_k (state after listing 1), coeff_out the
 * c_l.  Returns 0, 3 on an inexact division, 1 on overflow of `width`. */
int oracle_interp_listings(int n, const int64_t *x, const limb_t *y, size_t width,
                           limb_t *alpha_out, limb_t *coeff_out) {
    int saved = g_inexact;
    g_inexact = 0;
    bigint *c = (bigint *)xmalloc(sizeof(bigint) * (n + 1));
    for (int k = 0; k <= n; k++) c[k] = bi_from_twos(y + (size_t)k * width, width);
    listing_divided_differences(n, x, c);
    int ovf = 0;
    for (int k = 0; k <= n; k++) ovf |= bi_to_twos(&c[k], alpha_out + (size_t)k * width, width);
    listing_newton_to_monomial(n, x, c);
    for (int k = 0; k <= n; k++) ovf |= bi_to_twos(&c[k], coeff_out + (size_t)k * width, width);
    for (int k = 0; k <= n; k++) bi_free(&c[k]);
    free(c);
    int bad = g_inexact;
    g_inexact = saved || bad;
    return bad ? 3 : (ovf ? 1 : 0);
}

/* The even-odd driver of §4 (Eqs. 4.5-4.6) on given values:
 * y0 = W(0); yp[j] = W(2^j), ym[j] = W(-2^j), j = 0..n-1 (two's complement,
 * `width` limbs).  Writes w_0..w_{2n} to w_out.  Returns 0 / 3 / 1. */
int oracle_even_odd_interp(int n, const limb_t *y0, const limb_t *yp, const limb_t *ym,
                           size_t width, limb_t *w_out) {
    int saved = g_inexact;
    g_inexact = 0;
    bigint *We = (bigint *)xmalloc(sizeof(bigint) * (n + 1));
    bigint *Wo = (bigint *)xmalloc(sizeof(bigint) * (n + 1));
    int64_t *z = (int64_t *)xmalloc(sizeof(int64_t) * (n + 1));
    We[0] = bi_from_twos(y0, width);
    Wo[0] = bi_new(1);
    z[0] = 0;
    for (int j = 0; j < n; j++) {
        bigint a = bi_from_twos(yp + (size_t)j * width, width);
        bigint b = bi_from_twos(ym + (size_t)j * width, width);
        bigint s = bi_add(&a, &b);
        We[j + 1] = bi_divexact_word(&s, 2);
        bigint d = bi_sub(&a, &b);
        bigint dx = bi_shl(&d, (unsigned)j);
        Wo[j + 1] = bi_divexact_word(&dx, 2);
        z[j + 1] = (int64_t)1 << (2 * j);
        bi_free(&a); bi_free(&b); bi_free(&s); bi_free(&d); bi_free(&dx);
    }
    listing_divided_differences(n, z, We);
    listing_newton_to_monomial(n, z, We);
    listing_divided_differences(n, z, Wo);
    listing_newton_to_monomial(n, z, Wo);
    if (Wo[0].n != 0) g_inexact = 1;
    int ovf = 0;
    for (int k = 0; k <= 2 * n; k++) {
        const bigint *wk = (k % 2 == 0) ? &We[k / 2] : &Wo[(k - 1) / 2 + 1];
        ovf |= bi_to_twos(wk, w_out + (size_t)k * width, width);
    }
    for (int k = 0; k <= n; k++) { bi_free(&We[k]); bi_free(&Wo[k]); }
    free(We); free(Wo); free(z);
    int bad = g_inexact;
    g_inexact = saved || bad;
    return bad ? 3 : (ovf ? 1 : 0);
}

/* ------------------------------------------------------------------------- */
/* O3: residues                                                               */
/* ------------------------------------------------------------------------- */

/* a mod p by Horner from the top limb, p < 2^63. */
uint64_t oracle_mod(const limb_t *a, size_t n, uint64_t p) {
    unsigned __int128 r = 0;
    for (size_t i = n; i-- > 0;) {
        r = ((r << 32) | a[i]) % p;
    }
    return (uint64_t)r;
}

static uint64_t mulmod(uint64_t a, uint64_t b, uint64_t m) {
    return (uint64_t)(((unsigned __int128)a * b) % m);
}

static uint64_t powmod(uint64_t a, uint64_t e, uint64_t m) {
    uint64_t r = 1 % m;
    a %= m;
    while (e) {
        if (e & 1) r = mulmod(r, a, m);
        a = mulmod(a, a, m);
        e >>= 1;
    }
    return r;
}

/* Deterministic Miller-Rabin with the 12 prime bases 2..37 (exact for all
 * n < 3.18e23, in particular every 64-bit n). */
int oracle_is_prime_u64(uint64_t n) {
    static const uint64_t bases[12] = {2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37};
    if (n < 2) return 0;
    for (int i = 0; i < 12; i++) {
        if (n == bases[i]) return 1;
        if (n % bases[i] == 0) return 0;
    }
    uint64_t d = n - 1;
    int s = 0;
    while ((d & 1) == 0) { d >>= 1; s++; }
    for (int i = 0; i < 12; i++) {
        uint64_t x = powmod(bases[i], d, n);
        if (x == 1 || x == n - 1) continue;
        int comp = 1;
        for (int r = 1; r < s; r++) {
            x = mulmod(x, x, n);
            if (x == n - 1) { comp = 0; break; }
        }
        if (comp) return 0;
    }
    return 1;
}

/* α = log(2B-1)/log(B) (Eq. 2.3); used only in reports and as a pin. */
double oracle_alpha_exponent(int B) { return log(2.0 * B - 1.0) / log((double)B); }
