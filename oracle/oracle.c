/*
 * oracle.c -- plain, slow, obviously-correct CPU oracle for the hot path of
 * arXiv 2404.13216 (p-BiCGStab with ExBLAS-style exactly-rounded dots).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this code.  It
 * shares no source, header, table or helper with the CUDA library
 * (paper_2404_13216_b200/csrc); the two are independent implementations of
 * the same definitions.
 *
 * What it computes, and where that is defined:
 *
 *  EXDOT(x,y)  The binary64 nearest (ties-to-even) to the exact real
 *              sum_k x_k*y_k (the ExBLAS contract of
 *              PAPER.md §2 l.95: "independent of data partitioning, order of
 *              computations, thread scheduling, or reduction tree schemes").
 *              Computed by its definition: every product x_k*y_k is formed
 *              exactly as a 106-bit integer times 2^(ex+ey) and added into a
 *              big integer with LSB weight 2^-2148 (the exponent range of
 *              binary64 products); one rounding at the end.
 *              No floating-point expansion, no error-free transform.
 *              Range rule (reading R-9): a product with x,y != 0 and
 *              |fl(x*y)| < 2^-960 or |fl(x*y)| >= 2^1000 raises RANGE; the
 *              value stays exact.  NaN/Inf inputs raise NONFINITE.
 *
 *  SpMV        y_i = +0.0; for k over row i in ascending column order:
 *              y_i = fma(val_k, x[col_k], y_i)   (reading R-6).
 *
 *  p-BiCGStab  PAPER.md §2 Algorithm 2 (l.63-83) step by step, with the
 *              readings R-1..R-15 of DESIGN.md (w0 := A r0, scalar omega vs
 *              vector w, i=0 copies, FMA policy F, omega := 0 when (y,y)=0,
 *              relative breakdown thresholds, recursive-residual stopping).
 *              Range of its dots (R-9, R-24): full range (default
 *              of the Python binding): every dot is the exact sum rounded
 *              once over the whole binary64 range; only
 *              a NaN/Inf operand or an exact sum that rounds to +-inf stops
 *              the solve (RANGE).  Fast zone (range_mode 0, round 1's
 *              reading): any product outside the fast zone also stops it.
 *
 *  BiCGStab    PAPER.md §2 Algorithm 1 (l.39-54) in plain binary64 with
 *              sequential left-to-right dots (the "plain-double BiCGStab" of
 *              BASELINE.json north_star, used for the 1e-10 cross-check).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math (no x87, no
 * contraction: every a*b+c outside an explicit fma() is two roundings).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* --------------------------------------------------------------------------
 * Exact accumulator: two unsigned big integers (sum of positive products and
 * sum of magnitudes of negative products), 64-bit limbs, LSB weight 2^-2148.
 * 68 limbs = 4352 bits: products are < 2^2048, so 2^40 of them stay below
 * 2^2088 = bit 4236.
 * ------------------------------------------------------------------------ */
#define ORC_LIMBS 68
#define ORC_BIAS 2148 /* bit 0 has weight 2^-2148 */

enum { ORC_F_RANGE = 1, ORC_F_NONFINITE = 2, ORC_F_OVERFLOW = 4 /* the exact sum rounds to +-inf */ };

typedef struct {
    uint64_t pos[ORC_LIMBS];
    uint64_t neg[ORC_LIMBS];
    int flags;
} orc_acc;

void orc_acc_clear(orc_acc *a) { memset(a, 0, sizeof(*a)); }
int orc_acc_size(void) { return (int)sizeof(orc_acc); }
int orc_acc_flags(const orc_acc *a) { return a->flags; }

/* binary64 -> (integer mantissa m, exponent e) with |d| = m * 2^e exactly */
static void decompose(double d, uint64_t *m, int *e) {
    uint64_t bits;
    memcpy(&bits, &d, 8);
    int E = (int)((bits >> 52) & 0x7FF);
    uint64_t f = bits & ((1ULL << 52) - 1);
    if (E == 0) { *m = f; *e = -1074; }
    else { *m = f | (1ULL << 52); *e = E - 1075; }
}

/* add the 3-word value (w0,w1,w2) at limb index li into big integer v */
static void add_words(uint64_t *v, int li, uint64_t w0, uint64_t w1, uint64_t w2) {
    uint64_t w[3] = {w0, w1, w2};
    unsigned carry = 0;
    int i = li;
    for (int k = 0; k < 3 && i < ORC_LIMBS; ++k, ++i) {
        uint64_t s = v[i] + w[k];
        unsigned c1 = s < v[i];
        uint64_t s2 = s + carry;
        unsigned c2 = s2 < s;
        v[i] = s2;
        carry = c1 + c2;
    }
    while (carry && i < ORC_LIMBS) {
        v[i] += 1;
        carry = (v[i] == 0);
        ++i;
    }
}

/* acc += m * 2^e (m < 2^106 held in a 128-bit integer), sign s */
static void add_scaled(orc_acc *a, unsigned __int128 m, int e, int neg) {
    if (m == 0) return;
    int off = e + ORC_BIAS; /* >= 0 for every binary64 product */
    int li = off >> 6, sh = off & 63;
    uint64_t lo = (uint64_t)m, hi = (uint64_t)(m >> 64);
    uint64_t w0 = lo << sh;
    uint64_t w1 = (sh ? (lo >> (64 - sh)) : 0) | (hi << sh);
    uint64_t w2 = sh ? (hi >> (64 - sh)) : 0;
    add_words(neg ? a->neg : a->pos, li, w0, w1, w2);
}

/* acc += x*y exactly */
void orc_acc_add_product(orc_acc *a, double x, double y) {
    if (!isfinite(x) || !isfinite(y)) { a->flags |= ORC_F_NONFINITE; return; }
    if (x == 0.0 || y == 0.0) return;
    double p = x * y; /* only used for the range rule */
    if (fabs(p) < 0x1p-960 || fabs(p) >= 0x1p1000) a->flags |= ORC_F_RANGE;
    uint64_t mx, my;
    int ex, ey;
    decompose(x, &mx, &ex);
    decompose(y, &my, &ey);
    add_scaled(a, (unsigned __int128)mx * my, ex + ey, signbit(x) != signbit(y));
}

/* acc += x exactly (x is a binary64 value) */
void orc_acc_add_double(orc_acc *a, double x) {
    if (!isfinite(x)) { a->flags |= ORC_F_NONFINITE; return; }
    if (x == 0.0) return;
    uint64_t m;
    int e;
    decompose(x, &m, &e);
    add_scaled(a, m, e, signbit(x) != 0);
}

/* a += b exactly (merge of two partial accumulators) */
void orc_acc_merge(orc_acc *a, const orc_acc *b) {
    for (int s = 0; s < 2; ++s) {
        uint64_t *v = s ? a->neg : a->pos;
        const uint64_t *u = s ? b->neg : b->pos;
        unsigned carry = 0;
        for (int i = 0; i < ORC_LIMBS; ++i) {
            uint64_t t = v[i] + u[i];
            unsigned c1 = t < v[i];
            uint64_t t2 = t + carry;
            unsigned c2 = t2 < t;
            v[i] = t2;
            carry = c1 + c2;
        }
    }
    a->flags |= b->flags;
}

static int bit_of(const uint64_t *v, int i) { return (int)((v[i >> 6] >> (i & 63)) & 1); }

/* Round the exact value to the nearest binary64, ties to even. Exact zero
 * gives +0.0 (reading R-8).  Overflow gives +-inf and raises RANGE. */
double orc_acc_round(orc_acc *a) {
    uint64_t mag[ORC_LIMBS];
    int negative = 0;
    int cmp = 0;
    for (int i = ORC_LIMBS - 1; i >= 0 && cmp == 0; --i) {
        if (a->pos[i] > a->neg[i]) cmp = 1;
        else if (a->pos[i] < a->neg[i]) cmp = -1;
    }
    if (cmp == 0) return 0.0;
    const uint64_t *big = cmp > 0 ? a->pos : a->neg;
    const uint64_t *small = cmp > 0 ? a->neg : a->pos;
    negative = cmp < 0;
    unsigned borrow = 0;
    for (int i = 0; i < ORC_LIMBS; ++i) {
        uint64_t d = big[i] - small[i];
        unsigned b1 = big[i] < small[i];
        uint64_t d2 = d - borrow;
        unsigned b2 = d < (uint64_t)borrow;
        mag[i] = d2;
        borrow = b1 + b2;
    }
    int msb = -1;
    for (int i = ORC_LIMBS - 1; i >= 0; --i)
        if (mag[i]) { msb = i * 64 + 63 - __builtin_clzll(mag[i]); break; }
    int E = msb - ORC_BIAS; /* value in [2^E, 2^(E+1)) */
    if (E >= 1024) { a->flags |= ORC_F_RANGE | ORC_F_OVERFLOW; return negative ? -INFINITY : INFINITY; }
    int k = (E >= -1022) ? msb - 52 : (-1074 + ORC_BIAS); /* index of the kept LSB */
    uint64_t mant = 0;
    for (int i = msb; i >= k; --i) mant = (mant << 1) | (uint64_t)bit_of(mag, i);
    int round = (k >= 1) ? bit_of(mag, k - 1) : 0;
    int sticky = 0;
    for (int i = k - 2; i >= 0 && !sticky; --i) sticky = bit_of(mag, i);
    if (round && (sticky || (mant & 1))) {
        mant += 1;
        if (mant == (1ULL << 53)) { mant >>= 1; k += 1; }
    }
    double r = ldexp((double)mant, k - ORC_BIAS);
    if (isinf(r)) a->flags |= ORC_F_RANGE | ORC_F_OVERFLOW;
    return negative ? -r : r;
}

/* EXDOT(x,y); *flags receives ORC_F_* bits (may be NULL) */
double orc_exdot(int64_t n, const double *x, const double *y, int *flags) {
    orc_acc *a = (orc_acc *)malloc(sizeof(orc_acc));
    orc_acc_clear(a);
    for (int64_t k = 0; k < n; ++k) orc_acc_add_product(a, x[k], y[k]);
    double r = orc_acc_round(a);
    if (flags) *flags = a->flags;
    free(a);
    return r;
}

/* EXDOT computed as nparts contiguous blocks merged in the given order
 * (order: permutation of 0..nparts-1, or NULL for 0..nparts-1).  Used to
 * test partition/merge-order invariance. */
double orc_exdot_parts(int64_t n, const double *x, const double *y, int nparts, const int *order,
                       int *flags) {
    orc_acc *parts = (orc_acc *)malloc(sizeof(orc_acc) * (size_t)nparts);
    for (int p = 0; p < nparts; ++p) {
        orc_acc_clear(&parts[p]);
        int64_t s = n * p / nparts, e = n * (p + 1) / nparts;
        for (int64_t k = s; k < e; ++k) orc_acc_add_product(&parts[p], x[k], y[k]);
    }
    orc_acc *tot = (orc_acc *)malloc(sizeof(orc_acc));
    orc_acc_clear(tot);
    for (int p = 0; p < nparts; ++p) orc_acc_merge(tot, &parts[order ? order[p] : p]);
    double r = orc_acc_round(tot);
    if (flags) *flags = tot->flags;
    free(parts);
    free(tot);
    return r;
}

/* --------------------------------------------------------------------------
 * SpMV, fixed left-to-right per-row FMA chain (reading R-6)
 * ------------------------------------------------------------------------ */
void orc_spmv(int64_t nrows, const int32_t *rp, const int32_t *col, const double *val, const double *x,
              double *y) {
    for (int64_t i = 0; i < nrows; ++i) {
        double acc = +0.0;
        for (int32_t k = rp[i]; k < rp[i + 1]; ++k) acc = fma(val[k], x[col[k]], acc);
        y[i] = acc;
    }
}

/* y = Q x per 2x2 diagonal block (R-23): Q given as [nb][4]
 * row-major blocks over global rows (2m, 2m+1); y_2m = fma(q00, x_2m, q01 x_2m+1),
 * y_2m+1 = fma(q10, x_2m, q11 x_2m+1); the 1x1 tail block of an odd order:
 * y = q00 x.  (The C twin of oracle.bj_apply, pinned against it.) */
void orc_bj_apply(int64_t n, const double *Q, const double *x, double *y) {
    for (int64_t m = 0; 2 * m < n; ++m) {
        const double *q = Q + 4 * m;
        if (2 * m + 1 < n) {
            const double x0 = x[2 * m], x1 = x[2 * m + 1];
            y[2 * m] = fma(q[0], x0, q[1] * x1);
            y[2 * m + 1] = fma(q[2], x0, q[3] * x1);
        } else {
            y[2 * m] = q[0] * x[2 * m];
        }
    }
}

/* The 2x2 diagonal blocks of A and their inverses (R-23): rows
 * (2m, 2m+1), block (a b; c d), det = fma(a, d, -(b c)), M^-1 = (d -b; -c a)
 * / det with one RN division per entry; the 1x1 tail block of an odd order:
 * (a), 1/a.  M, Mi: [nb][4].  Returns 0, or 1 for a singular / non-finite
 * block.  (The C twin of oracle.block_jacobi_right's blocks, pinned against it.) */
static double csr_entry(const int32_t *rp, const int32_t *col, const double *val, int64_t r, int64_t c) {
    for (int32_t k = rp[r]; k < rp[r + 1]; ++k)
        if (col[k] == c) return val[k];
    return 0.0;
}
int orc_bj_blocks(int64_t n, const int32_t *rp, const int32_t *col, const double *val, double *M, double *Mi) {
    int bad = 0;
    for (int64_t m = 0; 2 * m < n; ++m) {
        const int64_t r0 = 2 * m;
        double *q = M + 4 * m, *qi = Mi + 4 * m;
        if (r0 + 1 < n) {
            const double a = csr_entry(rp, col, val, r0, r0), b = csr_entry(rp, col, val, r0, r0 + 1);
            const double c = csr_entry(rp, col, val, r0 + 1, r0), d = csr_entry(rp, col, val, r0 + 1, r0 + 1);
            const double det = fma(a, d, -(b * c));
            q[0] = a; q[1] = b; q[2] = c; q[3] = d;
            qi[0] = d / det; qi[1] = -(b / det); qi[2] = -(c / det); qi[3] = a / det;
            if (det == 0.0) bad = 1;
        } else {
            const double a = csr_entry(rp, col, val, r0, r0);
            q[0] = a; q[1] = 0.0; q[2] = 0.0; q[3] = 0.0;
            qi[0] = 1.0 / a; qi[1] = 0.0; qi[2] = 0.0; qi[3] = 0.0;
            if (a == 0.0) bad = 1;
        }
        for (int k = 0; k < 4; ++k)
            if (!isfinite(qi[k])) bad = 1;
    }
    return bad;
}

/* plain sequential fp64 dot (Algorithm 1 baseline; "Sequential") */
double orc_dot_seq(int64_t n, const double *x, const double *y) {
    double s = 0.0;
    for (int64_t k = 0; k < n; ++k) s = s + x[k] * y[k];
    return s;
}

/* --------------------------------------------------------------------------
 * p-BiCGStab (Algorithm 2), one iteration per orc_pbcg_step call.
 * ------------------------------------------------------------------------ */
enum { ORC_CONVERGED = 0, ORC_MAXITER = 1, ORC_BREAKDOWN_INIT = 2, ORC_BREAKDOWN_RHO = 3,
       ORC_BREAKDOWN_OMEGA = 4, ORC_BREAKDOWN_ALPHA = 5, ORC_RANGE = 6, ORC_RUNNING = -1 };
enum { ORC_OK = 0, ORC_EINVAL = 1, ORC_ENONFINITE = 5 };

/* history row layout (one row per iteration, row 0 = initialisation) */
enum { H_THETA = 0, H_ETA, H_SIGMA, H_ZETA, H_OMEGA, H_RHO, H_DELTA, H_RR, H_RELRES, H_BETA, H_ALPHA,
       H_COLS = 12 };

typedef struct {
    int64_t n;
    const int32_t *rp, *col;
    const double *val;
    double *b, *x, *r, *rh, *p, *s, *z, *q, *y, *w, *t, *v;
    double alpha, beta, omega, rho, sigma, zeta, nb, epsn, tol;
    int it, status, max_iter;
    double *hist; /* (max_iter+1)*H_COLS, caller-owned, may be NULL */
    double loop_seconds;
    int rr_period, replacements; /* residual replacement every rr_period iterations (0: never) */
    int full_range;              /* 1: only NONFINITE / OVERFLOW stop (R-24); 0: any RANGE flag stops (R-9) */
    const double *minv;          /* pipelined 2x2 block Jacobi (R-25): M^-1 blocks [nb][4], or NULL */
    double *tmp;                 /* M^-1 u scratch (n) */
} orc_pbcg;

/* The operator Algorithm 2 runs on: out = A u, or with the pipelined right
 * 2x2 block Jacobi preconditioner (R-25; PAPER.md l.90, l.93:
 * the preconditioner is applied inside the iteration) out = A (M^-1 u):
 * u_hat = M^-1 u by orc_bj_apply, then the per-row fma chain of A over u_hat. */
static void op_apply(orc_pbcg *S, const double *u, double *out) {
    if (S->minv) {
        orc_bj_apply(S->n, S->minv, u, S->tmp);
        orc_spmv(S->n, S->rp, S->col, S->val, S->tmp, out);
    } else {
        orc_spmv(S->n, S->rp, S->col, S->val, u, out);
    }
}

/* the flags of a dot phase that stop Algorithm 2 (R-9 / R-24) */
static int stops(const orc_pbcg *S, int f) {
    return S->full_range ? (f & (ORC_F_NONFINITE | ORC_F_OVERFLOW)) != 0 : f != 0;
}

int orc_pbcg_size(void) { return (int)sizeof(orc_pbcg); }

static double *vnew(int64_t n) { return (double *)calloc((size_t)(n > 0 ? n : 1), sizeof(double)); }

static int any_nonfinite(int64_t n, const double *v) {
    for (int64_t i = 0; i < n; ++i) if (!isfinite(v[i])) return 1;
    return 0;
}

static void hist_put(orc_pbcg *S, int row, int col, double v) {
    if (S->hist && row <= S->max_iter) S->hist[(int64_t)row * H_COLS + col] = v;
}

/* Lines I1-I4.  b == NULL means b := A*ones; x0 == NULL
 * means x0 := 0; full_range selects R-24 (1) or R-9 (0) for every dot;
 * minv != NULL: the iteration runs on B = A M^-1 applied as op_apply (R-25),
 * x0 is then the initial y0 = M x0 and x the final y (x = M^-1 y).  Returns ORC_OK / ORC_EINVAL / ORC_ENONFINITE; the solve
 * outcome is in S->status (ORC_RUNNING while iterations remain). */
int orc_pbcg_init(orc_pbcg *S, int64_t n, const int32_t *rp, const int32_t *col, const double *val,
                  const double *b, const double *x0, double tol, double eps, int max_iter, double *hist,
                  int full_range, const double *minv) {
    memset(S, 0, sizeof(*S));
    S->full_range = full_range != 0;
    S->minv = minv;
    S->n = n; S->rp = rp; S->col = col; S->val = val;
    S->tol = tol; S->max_iter = max_iter; S->hist = hist;
    if (n <= 0 || max_iter < 0 || !(tol >= 0.0)) return ORC_EINVAL;
    if (any_nonfinite(rp[n], val)) return ORC_ENONFINITE;
    S->b = vnew(n); S->x = vnew(n); S->r = vnew(n); S->rh = vnew(n); S->p = vnew(n);
    S->s = vnew(n); S->z = vnew(n); S->q = vnew(n); S->y = vnew(n); S->w = vnew(n);
    S->t = vnew(n); S->v = vnew(n); S->tmp = vnew(n);
    if (b) memcpy(S->b, b, sizeof(double) * (size_t)n);
    else {
        double *ones = vnew(n);
        for (int64_t i = 0; i < n; ++i) ones[i] = 1.0;
        orc_spmv(n, rp, col, val, ones, S->b);
        free(ones);
    }
    if (x0) memcpy(S->x, x0, sizeof(double) * (size_t)n);
    if (any_nonfinite(n, S->b) || any_nonfinite(n, S->x)) return ORC_ENONFINITE;
    /* I1: r0 := b - A x0 ; r^ := r0 ; w0 := A r0 ; t0 := A w0 */
    op_apply(S, S->x, S->v); /* v used as scratch for A x0 */
    for (int64_t i = 0; i < n; ++i) S->r[i] = S->b[i] - S->v[i];
    memset(S->v, 0, sizeof(double) * (size_t)n);
    memcpy(S->rh, S->r, sizeof(double) * (size_t)n);
    op_apply(S, S->r, S->w);
    op_apply(S, S->w, S->t);
    /* I2: norms and the first two inner products */
    int f0 = 0, f1 = 0, f2 = 0, f3 = 0;
    double bb = orc_exdot(n, S->b, S->b, &f0);
    S->nb = sqrt(bb);
    if (S->nb == 0.0) return ORC_EINVAL;
    double rho = orc_exdot(n, S->rh, S->r, &f1);
    double delta = orc_exdot(n, S->rh, S->w, &f2);
    double rr = orc_exdot(n, S->r, S->r, &f3);
    double relres = sqrt(rr) / S->nb;
    S->epsn = eps * sqrt(rho); /* eps * NORM(r^), with (r^,r^) = (r^,r0) = rho */
    S->rho = rho;
    hist_put(S, 0, H_RHO, rho);
    hist_put(S, 0, H_DELTA, delta);
    hist_put(S, 0, H_RR, rr);
    hist_put(S, 0, H_RELRES, relres);
    S->it = 0;
    if (stops(S, f0 | f1 | f2 | f3)) { S->status = ORC_RANGE; return ORC_OK; }
    /* I3 */
    if (relres <= tol) { S->status = ORC_CONVERGED; return ORC_OK; }
    /* I4: a0 := (r0,r0)/(r0,w0) */
    double a0 = rho / delta;
    if (delta == 0.0 || !isfinite(a0)) { S->status = ORC_BREAKDOWN_INIT; return ORC_OK; }
    S->alpha = a0;
    hist_put(S, 0, H_ALPHA, a0);
    S->status = (max_iter == 0) ? ORC_MAXITER : ORC_RUNNING;
    return ORC_OK;
}

/* One pass of the loop body of Algorithm 2. */
/* Residual replacement (§2 l.93: "resets the residuals r_i, along
 * with the auxiliary variables w_i, s_i, and z_i, to their original values
 * every k iterations"; SPEC.md l.246-249 adds t := A w for consistency).  At
 * the end of iteration i: r := b - A x (one rounding per entry, as r0),
 * w := A r, s := A p_i, z := A s, t := A w; scalars untouched.  v is left as
 * it is (R-21). */
int orc_pbcg_replace(orc_pbcg *S) {
    const int64_t n = S->n;
    double *ax = vnew(n);
    op_apply(S, S->x, ax);
    for (int64_t k = 0; k < n; ++k) S->r[k] = S->b[k] - ax[k];
    free(ax);
    op_apply(S, S->r, S->w);
    op_apply(S, S->p, S->s);
    op_apply(S, S->s, S->z);
    op_apply(S, S->w, S->t);
    S->replacements += 1;
    return ORC_OK;
}

void orc_pbcg_set_rr(orc_pbcg *S, int period) { S->rr_period = period > 0 ? period : 0; }
int orc_pbcg_replacements(const orc_pbcg *S) { return S->replacements; }

int orc_pbcg_step(orc_pbcg *S) {
    if (S->status != ORC_RUNNING) return S->status;
    struct timespec t0, t1;
    clock_gettime(CLOCK_MONOTONIC, &t0);
    const int64_t n = S->n;
    const int i = S->it;
    const double al = S->alpha, be = S->beta, om = S->omega;
    double *r = S->r, *p = S->p, *s = S->s, *z = S->z, *q = S->q, *y = S->y;
    double *w = S->w, *t = S->t, *v = S->v, *x = S->x, *rh = S->rh;
    /* S1 (l.70-72): p,s,z ; i = 0 uses beta_{-1} = 0 as exact copies (R-3) */
    if (i == 0) {
        memcpy(p, r, sizeof(double) * (size_t)n);
        memcpy(s, w, sizeof(double) * (size_t)n);
        memcpy(z, t, sizeof(double) * (size_t)n);
    } else {
        for (int64_t k = 0; k < n; ++k) {
            p[k] = fma(be, fma(-om, s[k], p[k]), r[k]); /* p := r + beta (p - omega s) */
            s[k] = fma(be, fma(-om, z[k], s[k]), w[k]); /* s := w + beta (s - omega z) */
            z[k] = fma(be, fma(-om, v[k], z[k]), t[k]); /* z := t + beta (z - omega v) */
        }
    }
    /* S2 (l.73-74) */
    for (int64_t k = 0; k < n; ++k) {
        q[k] = fma(-al, s[k], r[k]); /* q := r - alpha s */
        y[k] = fma(-al, z[k], w[k]); /* y := w - alpha z */
    }
    /* S3: phase-A inner products */
    int fA = 0, f;
    double theta = orc_exdot(n, q, y, &f); fA |= f;
    double eta = orc_exdot(n, y, y, &f); fA |= f;
    double sigma = orc_exdot(n, rh, s, &f); fA |= f;
    double zeta = orc_exdot(n, rh, z, &f); fA |= f;
    /* S4 (l.75): v := A z */
    op_apply(S, z, v);
    /* S5 (l.76): omega := (q,y)/(y,y), and 0 when (y,y) = 0 (R-12) */
    double omn = (eta == 0.0) ? 0.0 : theta / eta;
    hist_put(S, i + 1, H_THETA, theta);
    hist_put(S, i + 1, H_ETA, eta);
    hist_put(S, i + 1, H_SIGMA, sigma);
    hist_put(S, i + 1, H_ZETA, zeta);
    hist_put(S, i + 1, H_OMEGA, omn);
    if (stops(S, fA)) { S->status = ORC_RANGE; goto out; }
    /* S6 (l.77-79) */
    for (int64_t k = 0; k < n; ++k) {
        x[k] = fma(omn, q[k], fma(al, p[k], x[k]));   /* x := x + alpha p + omega q */
        r[k] = fma(-omn, y[k], q[k]);                 /* r := q - omega y */
        w[k] = fma(-omn, fma(-al, v[k], t[k]), y[k]); /* w := y - omega (t - alpha v) */
    }
    /* S7: phase-B inner products */
    int fB = 0;
    double rhon = orc_exdot(n, rh, r, &f); fB |= f;
    double deltan = orc_exdot(n, rh, w, &f); fB |= f;
    double rr = orc_exdot(n, r, r, &f); fB |= f;
    /* S8 (l.80): t := A w */
    op_apply(S, w, t);
    /* S9: recursive relative residual and the stopping rule (R-10) */
    double relres = sqrt(rr) / S->nb;
    hist_put(S, i + 1, H_RHO, rhon);
    hist_put(S, i + 1, H_DELTA, deltan);
    hist_put(S, i + 1, H_RR, rr);
    hist_put(S, i + 1, H_RELRES, relres);
    S->it = i + 1;
    S->omega = omn;
    if (stops(S, fB)) { S->status = ORC_RANGE; goto out; }
    if (relres <= S->tol) { S->status = ORC_CONVERGED; goto out; }
    /* S10: breakdown (R-11, R-12) */
    double thr = fmax(S->epsn * sqrt(rr), 1e-300);
    if (omn == 0.0) { S->status = ORC_BREAKDOWN_OMEGA; goto out; }
    if (fabs(rhon) <= thr) { S->status = ORC_BREAKDOWN_RHO; goto out; }
    /* S11 (l.81-82) */
    double ben = ((al / omn) * rhon) / S->rho;
    double d = fma(-(ben * omn), zeta, fma(ben, sigma, deltan));
    hist_put(S, i + 1, H_BETA, ben);
    /* S12 */
    if (!(fabs(d) > thr) || !isfinite(d)) { S->status = ORC_BREAKDOWN_ALPHA; goto out; }
    double aln = rhon / d;
    if (!isfinite(aln)) { S->status = ORC_BREAKDOWN_ALPHA; goto out; }
    hist_put(S, i + 1, H_ALPHA, aln);
    S->beta = ben;
    S->alpha = aln;
    S->rho = rhon;
    S->sigma = sigma;
    S->zeta = zeta;
    if (S->it >= S->max_iter) S->status = ORC_MAXITER;
    /* residual replacement (R-21) after every
     * rr_period-th completed iteration that leaves the solve running */
    if (S->status == ORC_RUNNING && S->rr_period > 0 && S->it % S->rr_period == 0) orc_pbcg_replace(S);
out:
    clock_gettime(CLOCK_MONOTONIC, &t1);
    S->loop_seconds += (double)(t1.tv_sec - t0.tv_sec) + 1e-9 * (double)(t1.tv_nsec - t0.tv_nsec);
    return S->status;
}

int orc_pbcg_run(orc_pbcg *S, int max_steps) {
    for (int k = 0; k < max_steps && S->status == ORC_RUNNING; ++k) orc_pbcg_step(S);
    return S->status;
}

/* true relative residual NORM(b - A x)/NORM(b) */
double orc_true_relres(int64_t n, const int32_t *rp, const int32_t *col, const double *val, const double *b,
                       const double *x, int *flags) {
    double *ax = vnew(n), *res = vnew(n);
    orc_spmv(n, rp, col, val, x, ax);
    for (int64_t i = 0; i < n; ++i) res[i] = b[i] - ax[i];
    int f1 = 0, f2 = 0;
    double rr = orc_exdot(n, res, res, &f1);
    double bb = orc_exdot(n, b, b, &f2);
    if (flags) *flags = f1 | f2;
    free(ax);
    free(res);
    return sqrt(rr) / sqrt(bb);
}

int orc_pbcg_iterations(const orc_pbcg *S) { return S->it; }
int orc_pbcg_status(const orc_pbcg *S) { return S->status; }
double orc_pbcg_loop_seconds(const orc_pbcg *S) { return S->loop_seconds; }
double orc_pbcg_scalar(const orc_pbcg *S, int which) {
    switch (which) {
    case 0: return S->alpha;
    case 1: return S->beta;
    case 2: return S->omega;
    case 3: return S->rho;
    case 4: return S->nb;
    case 5: return S->epsn;
    default: return NAN;
    }
}
/* vector access for tests: 0 b,1 x,2 r,3 rh,4 p,5 s,6 z,7 q,8 y,9 w,10 t,11 v */
const double *orc_pbcg_vec(const orc_pbcg *S, int which) {
    const double *tab[12] = {S->b, S->x, S->r, S->rh, S->p, S->s, S->z, S->q, S->y, S->w, S->t, S->v};
    return (which >= 0 && which < 12) ? tab[which] : NULL;
}
void orc_pbcg_free(orc_pbcg *S) {
    double *tab[12] = {S->b, S->x, S->r, S->rh, S->p, S->s, S->z, S->q, S->y, S->w, S->t, S->v};
    for (int k = 0; k < 12; ++k) free(tab[k]);
    free(S->tmp);
    memset(S, 0, sizeof(*S));
}

/* --------------------------------------------------------------------------
 * Plain-double BiCGStab, Algorithm 1 (l.39-54), sequential dots.
 * Returns status (ORC_CONVERGED / ORC_MAXITER / ORC_BREAKDOWN_*); x in/out.
 * Stopping rule: ||r_{i+1}||/||b|| <= tol (same rule as above); plus the
 * usual early exit when ||q_i||/||b|| <= tol (x := x + alpha p).
 * ------------------------------------------------------------------------ */
/* Algorithm 1 with the dot of the caller's choice:
 * exact = 0: sequential plain double (orc_dot_seq), the textbook routine the
 * north_star cross-check uses; exact = 1: EXDOT by its definition (orc_exdot)
 * -- the arithmetic the GPU's Alg. 1 arm reproduces bit for bit (SURVEY
 * §8(f) NEXT-1; R-20).  Everything else is the same code: -ffp-
 * contract=off, left-to-right evaluation as written below.  With exact dots
 * a product outside the exact zone (R-9) ends the solve with ORC_RANGE. */
static double a1_dot(int exact, int64_t n, const double *x, const double *y, int *flags) {
    if (!exact) return orc_dot_seq(n, x, y);
    int f = 0;
    const double v = orc_exdot(n, x, y, &f);
    *flags |= f;
    return v;
}

int orc_bicgstab_dots(int64_t n, const int32_t *rp, const int32_t *col, const double *val, const double *b,
                      double *x, double tol, int max_iter, int exact, int *iters, double *hist) {
    double *r = vnew(n), *rh = vnew(n), *p = vnew(n), *s = vnew(n), *q = vnew(n), *y = vnew(n);
    int status = ORC_MAXITER, it = 0, fl = 0;
    orc_spmv(n, rp, col, val, x, s);
    for (int64_t k = 0; k < n; ++k) r[k] = b[k] - s[k];
    memcpy(rh, r, sizeof(double) * (size_t)n);
    memcpy(p, r, sizeof(double) * (size_t)n);
    double nb = sqrt(a1_dot(exact, n, b, b, &fl));
    double rho = a1_dot(exact, n, rh, r, &fl);
    double rel = sqrt(a1_dot(exact, n, r, r, &fl)) / nb;
    if (hist) hist[0] = rel;
    if (fl) { status = ORC_RANGE; goto done; }
    if (rel <= tol) { status = ORC_CONVERGED; goto done; }
    for (int i = 0; i < max_iter; ++i) {
        orc_spmv(n, rp, col, val, p, s);                 /* s := A p */
        double den = a1_dot(exact, n, rh, s, &fl);
        if (fl) { status = ORC_RANGE; break; }
        if (den == 0.0) { status = ORC_BREAKDOWN_ALPHA; break; }
        double a = rho / den;                            /* a := (r0,r)/(r0,s) */
        for (int64_t k = 0; k < n; ++k) q[k] = r[k] - a * s[k];
        double qn = sqrt(a1_dot(exact, n, q, q, &fl)) / nb;
        if (fl) { status = ORC_RANGE; break; }
        if (qn <= tol) {
            for (int64_t k = 0; k < n; ++k) x[k] = x[k] + a * p[k];
            it = i + 1;
            if (hist) hist[it] = qn;
            status = ORC_CONVERGED;
            break;
        }
        orc_spmv(n, rp, col, val, q, y);                 /* y := A q */
        double yy = a1_dot(exact, n, y, y, &fl);
        double qy = a1_dot(exact, n, q, y, &fl);
        if (fl) { status = ORC_RANGE; break; }
        if (yy == 0.0) { status = ORC_BREAKDOWN_OMEGA; break; }
        double om = qy / yy;                             /* w := (q,y)/(y,y) */
        for (int64_t k = 0; k < n; ++k) {
            x[k] = x[k] + a * p[k] + om * q[k];
            r[k] = q[k] - om * y[k];
        }
        double rhon = a1_dot(exact, n, rh, r, &fl);
        it = i + 1;
        rel = sqrt(a1_dot(exact, n, r, r, &fl)) / nb;
        if (hist) hist[it] = rel;
        if (fl) { status = ORC_RANGE; break; }
        if (rel <= tol) { status = ORC_CONVERGED; break; }
        if (om == 0.0 || rho == 0.0 || rhon == 0.0) { status = ORC_BREAKDOWN_RHO; break; }
        double be = (a / om) * (rhon / rho);             /* beta := (a/w)(r0,r')/(r0,r) */
        for (int64_t k = 0; k < n; ++k) p[k] = r[k] + be * (p[k] - om * s[k]);
        rho = rhon;
    }
done:
    if (iters) *iters = it;
    free(r); free(rh); free(p); free(s); free(q); free(y);
    return status;
}

int orc_bicgstab(int64_t n, const int32_t *rp, const int32_t *col, const double *val, const double *b,
                 double *x, double tol, int max_iter, int *iters, double *hist) {
    return orc_bicgstab_dots(n, rp, col, val, b, x, tol, max_iter, 0, iters, hist);
}

