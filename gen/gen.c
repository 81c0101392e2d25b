/*
 * gen.c -- seeded synthetic inputs for the p-BiCGStab / ExBLAS hot path.
 *
 * INPUT GENERATORS ONLY.  This module is shared by the CPU oracle (oracle/),
 * the tests and bench.py, and it deliberately contains none of the method's
 * arithmetic: no SpMV, no dot products, no Krylov recurrences, no error-free
 * transforms, no superaccumulator.  It only builds matrices and vectors whose
 * shapes follow BASELINE.json `configs` (the stand-ins for the paper's
 * SuiteSparse test set, §3 l.103) as specified in SURVEY.md §8(d).
 *
 * PRNG: SplitMix64.  Every row (or vector element) draws from its own
 * substream keyed by (seed, index), so generation is embarrassingly parallel
 * and bit-identical for any thread count.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <quadmath.h>

#define GEN_VERSION 1

int gen_version(void) { return GEN_VERSION; }

/* ---------------------------------------------------------------- PRNG --- */
static inline uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
typedef struct { uint64_t s; } rng_t;
static inline rng_t rng_stream(uint64_t seed, uint64_t idx) {
    rng_t r;
    r.s = mix64(seed * 0x9E3779B97F4A7C15ULL + 0x632BE59BD9B4E019ULL) ^ mix64(idx + 0xD1B54A32D192ED03ULL);
    return r;
}
static inline uint64_t rng_u64(rng_t *r) {
    r->s += 0x9E3779B97F4A7C15ULL;
    return mix64(r->s);
}
/* 53-bit uniform in [0,1) */
static inline double rng_unif(rng_t *r) { return (double)(rng_u64(r) >> 11) * 0x1.0p-53; }

/* ------------------------------------------------ convection-diffusion --- */
/*
 * -Lap(u) + c.grad(u), c = (Pe,...,Pe), homogeneous Dirichlet, N interior
 * points per axis, h = 1/(N+1), first-order upwind (backward differences
 * since c > 0), rows scaled by h^2:
 *     lower neighbours (-x,-y,-z): -(1 + h*Pe)
 *     upper neighbours (+x,+y,+z): -1
 *     diagonal                   : 2d + d*h*Pe
 * Row index r = i + N*j (+ N^2*k), x fastest; columns strictly ascending.
 * BASELINE.json configs[0] (d=2,N=64,Pe=10), [2] (d=3,N=128,Pe=100),
 * [4] (d=3,N=256,Pe=200).
 */
int64_t gen_stencil_nnz(int d, int64_t N) {
    int64_t n = 1, nd1 = 1;
    for (int a = 0; a < d; ++a) n *= N;
    for (int a = 0; a < d - 1; ++a) nd1 *= N;
    return (2 * d + 1) * n - 2 * d * nd1;
}

int gen_stencil(int d, int64_t N, double Pe, int32_t *row_ptr, int32_t *col, double *val) {
    if (d != 2 && d != 3) return 1;
    const double h = 1.0 / (double)(N + 1);
    const double hc = h * Pe;
    const double lo = -(1.0 + hc);
    const double up = -1.0;
    const double dg = (double)(2 * d) + (double)d * hc;
    int64_t n = (d == 2) ? N * N : N * N * N;
    int64_t NN = N * N;
    /* row lengths are analytic, so fill in parallel from a closed-form prefix */
    row_ptr[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        int64_t i = r % N, j = (r / N) % N, k = (d == 3) ? r / NN : 0;
        int len = 1 + (i > 0) + (i < N - 1) + (j > 0) + (j < N - 1);
        if (d == 3) len += (k > 0) + (k < N - 1);
        row_ptr[r + 1] = (int32_t)(row_ptr[r] + len);
    }
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
        int64_t i = r % N, j = (r / N) % N, k = (d == 3) ? r / NN : 0;
        int64_t p = row_ptr[r];
        if (d == 3 && k > 0)     { col[p] = (int32_t)(r - NN); val[p++] = lo; }
        if (j > 0)               { col[p] = (int32_t)(r - N);  val[p++] = lo; }
        if (i > 0)               { col[p] = (int32_t)(r - 1);  val[p++] = lo; }
        col[p] = (int32_t)r; val[p++] = dg;
        if (i < N - 1)           { col[p] = (int32_t)(r + 1);  val[p++] = up; }
        if (j < N - 1)           { col[p] = (int32_t)(r + N);  val[p++] = up; }
        if (d == 3 && k < N - 1) { col[p] = (int32_t)(r + NN); val[p++] = up; }
    }
    return 0;
}

/* ------------------------------------------------ random banded (C4) ---- */
/*
 * BASELINE.json configs[3]: row length L = clip(Poisson(lambda), lmin, lmax)
 * including the diagonal; L-1 distinct off-diagonal columns uniform in
 * [r-band, r+band] \ {r} clipped to [0,n), sorted; off-diagonal values N(0,1)
 * (Box-Muller); diagonal = diag_scale * (left-to-right sum of |off-diag|).
 * Draw order per row substream (seed,row): L, then columns, then values.
 */
static int poisson_draw(rng_t *r, double lambda) {
    double u = rng_unif(r);
    double p = exp(-lambda), cdf = p;
    int k = 0;
    while (u > cdf && k < 100000) {
        k += 1;
        p *= lambda / (double)k;
        cdf += p;
        if (p == 0.0) break;
    }
    return k;
}
static int row_len_draw(rng_t *r, double lambda, int lmin, int lmax, int64_t avail) {
    int L = poisson_draw(r, lambda);
    if (L < lmin) L = lmin;
    if (L > lmax) L = lmax;
    if ((int64_t)L - 1 > avail) L = (int)(avail + 1);
    return L;
}

int gen_random_rowlens(int64_t n, uint64_t seed, double lambda, int lmin, int lmax, int64_t band,
                       int32_t *row_ptr) {
    int32_t *len = (int32_t *)malloc(sizeof(int32_t) * (size_t)n);
    if (!len) return 2;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < n; ++r) {
        rng_t g = rng_stream(seed, (uint64_t)r);
        int64_t lo = r - band < 0 ? 0 : r - band;
        int64_t hi = r + band > n - 1 ? n - 1 : r + band;
        len[r] = row_len_draw(&g, lambda, lmin, lmax, hi - lo);
    }
    int64_t acc = 0;
    row_ptr[0] = 0;
    for (int64_t r = 0; r < n; ++r) {
        acc += len[r];
        if (acc > INT32_MAX) { free(len); return 3; }
        row_ptr[r + 1] = (int32_t)acc;
    }
    free(len);
    return 0;
}

int gen_random_fill(int64_t n, uint64_t seed, double lambda, int lmin, int lmax, int64_t band,
                    double diag_scale, const int32_t *row_ptr, int32_t *col, double *val) {
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : bad)
    for (int64_t r = 0; r < n; ++r) {
        rng_t g = rng_stream(seed, (uint64_t)r);
        int64_t lo = r - band < 0 ? 0 : r - band;
        int64_t hi = r + band > n - 1 ? n - 1 : r + band;
        int L = row_len_draw(&g, lambda, lmin, lmax, hi - lo);
        if (L != row_ptr[r + 1] - row_ptr[r]) { bad |= 1; continue; }
        int32_t c[1024];
        double v[1024];
        if (L > 1024) { bad |= 1; continue; }
        int m = 0;
        while (m < L - 1) { /* rejection sampling of distinct off-diagonal columns */
            int64_t cc = lo + (int64_t)(rng_unif(&g) * (double)(hi - lo + 1));
            if (cc > hi) cc = hi;
            if (cc == r) continue;
            int dup = 0;
            for (int q = 0; q < m; ++q) if (c[q] == cc) { dup = 1; break; }
            if (dup) continue;
            c[m++] = (int32_t)cc;
        }
        for (int a = 1; a < m; ++a) { /* insertion sort */
            int32_t t = c[a]; int b = a - 1;
            while (b >= 0 && c[b] > t) { c[b + 1] = c[b]; --b; }
            c[b + 1] = t;
        }
        for (int q = 0; q < m; ++q) { /* Box-Muller N(0,1) */
            double u1 = 1.0 - rng_unif(&g), u2 = rng_unif(&g);
            v[q] = sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2);
        }
        double asum = 0.0;
        for (int q = 0; q < m; ++q) asum = asum + fabs(v[q]);
        double dgv = diag_scale * asum;
        if (dgv == 0.0) dgv = 1.0;
        int64_t p = row_ptr[r];
        int placed = 0;
        for (int q = 0; q < m; ++q) {
            if (!placed && c[q] > r) { col[p] = (int32_t)r; val[p++] = dgv; placed = 1; }
            col[p] = c[q]; val[p++] = v[q];
        }
        if (!placed) { col[p] = (int32_t)r; val[p++] = dgv; }
    }
    return bad ? 4 : 0;
}

/* ----------------------------------------------------------- vectors ---- */
/* u in [lo,hi): v_k = lo + (hi-lo)*u_k, substream (seed,k) */
int gen_uniform(int64_t n, uint64_t seed, double lo, double hi, double *v) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) {
        rng_t g = rng_stream(seed, (uint64_t)k);
        v[k] = lo + (hi - lo) * rng_unif(&g);
    }
    return 0;
}

/*
 * Ill-conditioned dot-product pairs, Ogita-Rump-Oishi GenDot style
 * (BASELINE.json configs[1]), built block-wise so
 * that 2^28-element vectors generate in seconds:
 *   for each block of `blk` elements (substream (seed, block)):
 *   1. b = log2 target condition (~100 for cond 1e30);
 *   2. first half: random mantissas/signs, exponents uniform in [0,b/2]
 *      (first one pinned to b/2, last one to 0);
 *   3. second half: exponents falling linearly from b/2 to 0, and
 *      y_k = (u*2^e_k - D_{k-1}) / x_k with D the block's running dot, tracked
 *      in binary128 (a generator-local approximation; the achieved condition
 *      of the whole vector is measured afterwards by the oracle);
 *   4. Fisher-Yates shuffle inside the block;
 *   5. global scale 2^-25 on x and y, then reciprocal power-of-two shifts
 *      x_k*2^s_k, y_k*2^-s_k with s_k uniform in [-spread,spread] (products and
 *      the dot are unchanged up to the exact 2^-50 factor).
 * Blocks are independent, each nearly cancels, so the condition of the
 * concatenation is about sqrt(#blocks) times a block's.
 */
static void gendot_block(int64_t m, uint64_t seed, uint64_t blk_id, double b, int spread,
                         double *x, double *y) {
    rng_t g = rng_stream(seed, 0x100000000ull + blk_id);
    const double half = 0.5 * b;
    int64_t n2 = m / 2;
    for (int64_t k = 0; k < n2; ++k) {
        double e = (k == 0) ? half : (k == n2 - 1) ? 0.0 : floor(rng_unif(&g) * (half + 1.0));
        if (e > half) e = half;
        x[k] = ldexp(2.0 * rng_unif(&g) - 1.0, (int)e);
        y[k] = ldexp(2.0 * rng_unif(&g) - 1.0, (int)e);
    }
    __float128 D = 0;
    for (int64_t k = 0; k < n2; ++k) D += (__float128)x[k] * (__float128)y[k];
    for (int64_t k = n2; k < m; ++k) {
        double t = (m - n2 > 1) ? (double)(k - n2) / (double)(m - n2 - 1) : 1.0;
        int e = (int)floor(half * (1.0 - t) + 0.5);
        double xk = ldexp(2.0 * rng_unif(&g) - 1.0, e);
        if (xk == 0.0) xk = ldexp(1.0, e);
        double target = ldexp(2.0 * rng_unif(&g) - 1.0, e);
        double yk = (target - (double)D) / xk;
        x[k] = xk;
        y[k] = yk;
        D += (__float128)xk * (__float128)yk;
    }
    for (int64_t k = m - 1; k > 0; --k) {
        int64_t j = (int64_t)(rng_unif(&g) * (double)(k + 1));
        if (j > k) j = k;
        double tx = x[k]; x[k] = x[j]; x[j] = tx;
        double ty = y[k]; y[k] = y[j]; y[j] = ty;
    }
    for (int64_t k = 0; k < m; ++k) {
        int s = spread ? (int)(rng_u64(&g) % (uint64_t)(2 * spread + 1)) - spread : 0;
        x[k] = ldexp(x[k], s - 25);
        y[k] = ldexp(y[k], -s - 25);
    }
}

int gen_ill(int64_t n, uint64_t seed, double b, int spread, int64_t blk, double *x, double *y) {
    if (n < 4) return 1;
    if (blk < 4) blk = n;
    int64_t nb = (n + blk - 1) / blk;
#pragma omp parallel for schedule(dynamic, 1)
    for (int64_t q = 0; q < nb; ++q) {
        int64_t s = q * blk, e = s + blk < n ? s + blk : n;
        gendot_block(e - s, seed, (uint64_t)q, b, spread, x + s, y + s);
    }
    return 0;
}

/* log-uniform magnitudes in [2^emin, 2^emax) with random signs (tests) */
int gen_loguniform(int64_t n, uint64_t seed, double emin, double emax, double *v) {
#pragma omp parallel for schedule(static)
    for (int64_t k = 0; k < n; ++k) {
        rng_t g = rng_stream(seed, (uint64_t)k);
        double e = emin + (emax - emin) * rng_unif(&g);
        double m = 1.0 + rng_unif(&g);
        double s = (rng_u64(&g) >> 63) ? -1.0 : 1.0;
        v[k] = s * ldexp(m, (int)floor(e));
    }
    return 0;
}
