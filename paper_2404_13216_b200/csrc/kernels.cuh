// kernels.cuh -- the sm_100a kernels of the p-BiCGStab + ExBLAS hot path.
//
//   phase_finalize   the scalar steps of Alg. 2 (and Alg. 1) from rounded dots
//   multidot         generic fused EXDOTs (init, true residual, Alg. 1 phases)
//   finalize         normalise + round + scalars (side stream / after allreduce)
//   spmv_sell[_pipe] l.75 v = A z, l.80 t = A w: per-row ordered FMA chain on a
//                    sliced-ELL (C = 32) layout         [a5, a10; reading R-6]
//   a1_*, plain_*    the Alg. 1 and plain-dot arms
//   setup helpers    SELL conversion, slot records, Jacobi scaling
// The K2/K3 recurrences + dots, the EXDOT stream and the packed SELL-P SpMV
// are the TMA kernels of stream.cuh.
//
// Every floating-point value op is an explicit __fma_rn/__dmul_rn/__dadd_rn or
// an IEEE division/sqrt; the library is compiled with -fmad=false.
#pragma once
#include <cstdint>

#include "exblas.cuh"

namespace pbcg {

// history row layout (identical to the oracle's, include/pbicgstab.h)
enum { H_THETA = 0, H_ETA, H_SIGMA, H_ZETA, H_OMEGA, H_RHO, H_DELTA, H_RR, H_RELRES, H_BETA, H_ALPHA, H_COLS = 12 };
enum { ST_CONVERGED = 0, ST_MAXITER = 1, ST_BD_INIT = 2, ST_BD_RHO = 3, ST_BD_OMEGA = 4, ST_BD_ALPHA = 5,
       ST_RANGE = 6, ST_RUNNING = -1 };
enum Phase { PH_INIT = 0, PH_A = 1, PH_B = 2, PH_TRUE = 3, PH_EXDOT = 4,
             // I2-I4 when x0 = 0, so r0 = r^ = b bit for bit: two dots, (w0,b) = (r^,w0) and (b,b) =
             // (b,b) = (r^,r0) = (r0,r0)
             PH_INIT0 = 5,
             // Algorithm 1 (classic BiCGStab, reading R-20)
             PH1_INIT = 6, PH1_DEN = 7, PH1_QQ = 8, PH1_OM = 9, PH1_R = 10 };

// device-resident solver scalars (one copy per rank; identical on all ranks)
struct Scalars {
    double alpha, beta, omega, rho, sigma, zeta;
    double nb, epsn, tol, eps;
    double relres, relres_true;
    int32_t it, done, status, max_iter;
    int32_t hist_cap, err;
    int32_t qconv;  // Alg. 1: converged at the q check, x += alpha p still to apply
    int32_t range_mode;  // Alg. 2 dots: 0 full range (R-24: corrected, only NaN/Inf or overflow stop), 1 fast zone (R-9)
    unsigned long long digest;  // pbcg_result.digest of the history rows (hist_digest_kernel, at finish)
};

// ------------------------------------------------------------------------
// phase finalisation (one thread): the scalar part of Algorithm 2
// ------------------------------------------------------------------------
__device__ __forceinline__ void hist_put(double *hist, const Scalars *sc, int row, int col, double v) {
    if (hist && row < sc->hist_cap) hist[(int64_t)row * H_COLS + col] = v;
}

// Algorithm 1 with exact dots: the scalar steps of the oracle's
// orc_bicgstab_dots (exact = 1) in the same order (reading R-20).
__device__ void phase1_finalize(int phase, Scalars *sc, const double *d, unsigned flags, double *hist) {
    if (phase == PH1_INIT) {  // nb, rho0 = (r^,r0), relres0
        const double bb = d[0], rho = d[1], rr = d[2];
        sc->it = 0;
        sc->nb = __dsqrt_rn(bb);
        if (sc->nb == 0.0) { sc->err = 1; sc->done = 1; sc->status = ST_MAXITER; return; }  // EINVAL
        const double rel = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
        sc->rho = rho;
        sc->relres = rel;
        hist_put(hist, sc, 0, H_RHO, rho);
        hist_put(hist, sc, 0, H_RELRES, rel);
        if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
        if (rel <= sc->tol) { sc->status = ST_CONVERGED; sc->done = 1; return; }
        if (sc->max_iter == 0) { sc->status = ST_MAXITER; sc->done = 1; return; }
        sc->status = ST_RUNNING;
        return;
    }
    if (sc->done) return;
    const int i = sc->it;
    if (phase == PH1_DEN) {  // a := (r0,r)/(r0,s)
        if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
        if (d[0] == 0.0) { sc->status = ST_BD_ALPHA; sc->done = 1; return; }
        sc->alpha = __ddiv_rn(sc->rho, d[0]);
        hist_put(hist, sc, i + 1, H_ALPHA, sc->alpha);
        return;
    }
    if (phase == PH1_QQ) {  // early exit on ||q||/||b|| <= tol: x := x + a p, done
        const double qn = __ddiv_rn(__dsqrt_rn(d[0]), sc->nb);
        if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
        if (qn <= sc->tol) {
            sc->it = i + 1;
            sc->relres = qn;
            hist_put(hist, sc, i + 1, H_RELRES, qn);
            sc->status = ST_CONVERGED;
            sc->qconv = 1;
            sc->done = 1;
        }
        return;
    }
    if (phase == PH1_OM) {  // w := (q,y)/(y,y)
        const double qy = d[0], yy = d[1];
        if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
        if (yy == 0.0) { sc->status = ST_BD_OMEGA; sc->done = 1; return; }
        sc->omega = __ddiv_rn(qy, yy);
        hist_put(hist, sc, i + 1, H_OMEGA, sc->omega);
        return;
    }
    // PH1_R: rho' = (r0,r'), relres; stopping; beta := (a/w)(rho'/rho)
    const double rhon = d[0], rr = d[1];
    const double rel = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
    sc->it = i + 1;
    sc->relres = rel;
    hist_put(hist, sc, i + 1, H_RHO, rhon);
    hist_put(hist, sc, i + 1, H_RR, rr);
    hist_put(hist, sc, i + 1, H_RELRES, rel);
    if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
    if (rel <= sc->tol) { sc->status = ST_CONVERGED; sc->done = 1; return; }
    const double om = sc->omega;
    if (om == 0.0 || sc->rho == 0.0 || rhon == 0.0) { sc->status = ST_BD_RHO; sc->done = 1; return; }
    const double be = __dmul_rn(__ddiv_rn(sc->alpha, om), __ddiv_rn(rhon, sc->rho));
    hist_put(hist, sc, i + 1, H_BETA, be);
    sc->beta = be;
    sc->rho = rhon;
    if (sc->it >= sc->max_iter) { sc->status = ST_MAXITER; sc->done = 1; }
}

__device__ void phase_finalize(int phase, Scalars *sc, const double *d, unsigned flags, double *hist,
                               double *out, int32_t *out_flags) {
    if (phase >= PH1_INIT) {
        phase1_finalize(phase, sc, d, flags, hist);
        return;
    }
    if (phase == PH_EXDOT) {
        if (out) *out = d[0];
        if (out_flags) *out_flags = (int32_t)flags;
        return;
    }
    if (phase == PH_TRUE) {  // NORM(b - A x)/NORM(b)
        sc->relres_true = __ddiv_rn(__dsqrt_rn(d[0]), sc->nb);
        return;
    }
    if (phase == PH_INIT || phase == PH_INIT0) {  // lines I2-I4
        const double bb = phase == PH_INIT ? d[0] : d[1], rho = phase == PH_INIT ? d[1] : d[1],
                     delta = phase == PH_INIT ? d[2] : d[0], rr = phase == PH_INIT ? d[3] : d[1];
        sc->it = 0;
        sc->nb = __dsqrt_rn(bb);
        if (sc->nb == 0.0) { sc->err = 1; sc->done = 1; sc->status = ST_MAXITER; return; }  // EINVAL
        const double relres = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
        sc->epsn = __dmul_rn(sc->eps, __dsqrt_rn(rho));  // eps * NORM(r^), (r^,r^) = (r^,r0) = rho
        sc->rho = rho;
        sc->relres = relres;
        hist_put(hist, sc, 0, H_RHO, rho);
        hist_put(hist, sc, 0, H_DELTA, delta);
        hist_put(hist, sc, 0, H_RR, rr);
        hist_put(hist, sc, 0, H_RELRES, relres);
        if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
        if (relres <= sc->tol) { sc->status = ST_CONVERGED; sc->done = 1; return; }
        const double a0 = __ddiv_rn(rho, delta);
        if (delta == 0.0 || !isfinite(a0)) { sc->status = ST_BD_INIT; sc->done = 1; return; }
        sc->alpha = a0;
        hist_put(hist, sc, 0, H_ALPHA, a0);
        if (sc->max_iter == 0) { sc->status = ST_MAXITER; sc->done = 1; return; }
        sc->status = ST_RUNNING;
        return;
    }
    if (phase == PH_A) {  // l.76: omega := (q,y)/(y,y); omega := 0 when (y,y) = 0 (R-12)
        const int i = sc->it;
        const double theta = d[0], eta = d[1], sigma = d[2], zeta = d[3];
        const double om = (eta == 0.0) ? 0.0 : __ddiv_rn(theta, eta);
        hist_put(hist, sc, i + 1, H_THETA, theta);
        hist_put(hist, sc, i + 1, H_ETA, eta);
        hist_put(hist, sc, i + 1, H_SIGMA, sigma);
        hist_put(hist, sc, i + 1, H_ZETA, zeta);
        hist_put(hist, sc, i + 1, H_OMEGA, om);
        if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
        sc->omega = om;
        sc->sigma = sigma;
        sc->zeta = zeta;
        return;
    }
    // PH_B: l.81-82 and the stopping / breakdown rules (R-10, R-11)
    const int i = sc->it;
    const double rhon = d[0], deltan = d[1], rr = d[2];
    const double relres = __ddiv_rn(__dsqrt_rn(rr), sc->nb);
    hist_put(hist, sc, i + 1, H_RHO, rhon);
    hist_put(hist, sc, i + 1, H_DELTA, deltan);
    hist_put(hist, sc, i + 1, H_RR, rr);
    hist_put(hist, sc, i + 1, H_RELRES, relres);
    sc->it = i + 1;
    sc->relres = relres;
    if (flags) { sc->status = ST_RANGE; sc->done = 1; return; }
    if (relres <= sc->tol) { sc->status = ST_CONVERGED; sc->done = 1; return; }
    const double thr = fmax(__dmul_rn(sc->epsn, __dsqrt_rn(rr)), 1e-300);
    const double om = sc->omega, al = sc->alpha;
    if (om == 0.0) { sc->status = ST_BD_OMEGA; sc->done = 1; return; }
    if (fabs(rhon) <= thr) { sc->status = ST_BD_RHO; sc->done = 1; return; }
    const double ben = __ddiv_rn(__dmul_rn(__ddiv_rn(al, om), rhon), sc->rho);  // ((a/w) rho')/rho
    const double dd = __fma_rn(-__dmul_rn(ben, om), sc->zeta, __fma_rn(ben, sc->sigma, deltan));
    hist_put(hist, sc, i + 1, H_BETA, ben);
    if (!(fabs(dd) > thr) || !isfinite(dd)) { sc->status = ST_BD_ALPHA; sc->done = 1; return; }
    const double aln = __ddiv_rn(rhon, dd);
    if (!isfinite(aln)) { sc->status = ST_BD_ALPHA; sc->done = 1; return; }
    hist_put(hist, sc, i + 1, H_ALPHA, aln);
    sc->beta = ben;
    sc->alpha = aln;
    sc->rho = rhon;
    if (sc->it >= sc->max_iter) { sc->status = ST_MAXITER; sc->done = 1; }
}

// ------------------------------------------------------------------------
// Full-range EXDOT (closes reading R-9 for exdot).  The
// fast kernels are exact for every product whose TwoProd is exact; a product
// outside that zone raises FLAG_RANGE.  In a standalone single-GPU dot, each
// CTA that raised it corrects ITS OWN flagged products (cta_full_range): the
// exact product -- the 106-bit integer mx*my times 2^(ex+ey), ex+ey >= -2148
// -- minus what its FPE received, into an extended superaccumulator of XS_L
// 32-bit digits with LSB weight 2^-2148 (the binary64 product range),
// normalised and added into gacc[XS_OFF ..].  The last CTA adds the fast
// words (2^-1074 = extended bit 1074) and rounds once (RN-even, subnormals,
// overflow to +-inf).  Only the flagged CTAs pay, in parallel.
// ------------------------------------------------------------------------
constexpr int XS_L = 136;   // 4352 bits: 2^-2148 .. 2^2204 (products < 2^2048, sums of < 2^40 of them)
// word layout of an ND-dot reduction buffer: ND * SACC_L fast words, the
// SACC_FLAGW flag counts, padding, then ND extended accumulators of XS_L words
// (written only by CTAs that met a product outside the fast zone)
__host__ __device__ constexpr int xs_off(int nd) { return ((nd * SACC_L + SACC_FLAGW + 7) / 8) * 8; }
__host__ __device__ constexpr int xs_words(int nd) { return xs_off(nd) + nd * XS_L; }
constexpr int XS_OFF = xs_off(1);     // 72: the standalone EXDOT's extended accumulator
constexpr int XS_GW = xs_words(1);    // gacc words a full-range EXDOT needs

__device__ __forceinline__ void dbl_parts(double v, unsigned long long &m, int &e) {
    const unsigned long long b = (unsigned long long)__double_as_longlong(v);
    const int E = (int)((b >> 52) & 0x7FF);
    m = b & 0xFFFFFFFFFFFFFull;
    if (E) { m |= 1ull << 52; e = E - 1075; } else { e = -1074; }
}

// the exact product a*b (finite) into the shared extended accumulator
__device__ __forceinline__ void xs_add_product(unsigned long long *X, double a, double b) {
    if (a == 0.0 || b == 0.0) return;
    unsigned long long ma, mb;
    int ea, eb;
    dbl_parts(a, ma, ea);
    dbl_parts(b, mb, eb);
    const unsigned long long lo = ma * mb, hi = __umul64hi(ma, mb);  // the 106-bit product
    const int off = ea + eb + 2148;                                    // >= 0
    const int w = off >> 5, sh = off & 31;
    const unsigned long long l2 = lo << sh;
    const unsigned long long h2 = (hi << sh) | (sh ? (lo >> (64 - sh)) : 0ull);
    const unsigned long long top = sh ? (hi >> (64 - sh)) : 0ull;
    const long long d[5] = {(long long)(l2 & 0xFFFFFFFFull), (long long)(l2 >> 32), (long long)(h2 & 0xFFFFFFFFull),
                            (long long)(h2 >> 32), (long long)top};
    const bool neg = (a < 0.0) != (b < 0.0);
#pragma unroll
    for (int j = 0; j < 5; ++j)
        if (d[j]) sacc_add_shared(&X[w + j], neg ? -d[j] : d[j]);
}

// carry-propagate XS_L signed digits into [0, 2^32) (top word signed); one thread
__device__ __forceinline__ void xs_normalize(long long *wd) {
    long long carry = 0;
    for (int i = 0; i < XS_L - 1; ++i) {
        const long long v = wd[i] + carry;
        carry = v >> 32;
        wd[i] = v & 0xFFFFFFFFll;
    }
    wd[XS_L - 1] += carry;
}

// round the normalised extended value once (RN-even, subnormals, +-inf); one thread
__device__ double xs_round(long long *wd) {
    const bool neg = wd[XS_L - 1] < 0;
    if (neg) {  // magnitude (two's complement negation over the digits)
        unsigned long long c = 1;
        for (int i = 0; i < XS_L; ++i) {
            const unsigned long long v = (unsigned long long)(~(unsigned)wd[i]) + c;
            wd[i] = (long long)(v & 0xFFFFFFFFull);
            c = v >> 32;
        }
    }
    int t = -1;  // highest set bit
    for (int i = XS_L - 1; i >= 0 && t < 0; --i)
        if (wd[i]) t = 32 * i + 31 - __clz((unsigned)wd[i]);
    double r = 0.0;
    if (t >= 0) {
        auto bit = [&](int k) -> unsigned { return k < 0 ? 0u : (unsigned)(wd[k >> 5] >> (k & 31)) & 1u; };
        const int q = max(t - 52, 1074);  // the result's LSB: 53 bits, or the subnormal quantum 2^-1074
        unsigned long long M = 0;
        for (int k = t; k >= q; --k) M = (M << 1) | bit(k);
        const unsigned half = bit(q - 1);
        bool sticky = false;
        for (int k = q - 2; k >= 0 && !sticky; --k) sticky = bit(k) != 0u;
        if (half && (sticky || (M & 1ull))) ++M;
        r = scalbn((double)M, q - 2148);  // exact, or +inf on overflow
        if (neg) r = -r;
    }
    return r;
}

// A CTA whose fast pass raised a flag, at its end (all threads; S.flags holds
// the CTA's flags).  Its elements are read once more: a NaN/Inf input makes
// the dot non-finite; a flagged product of finite operands
// had entered the FPE as p + e with e inexact (|x y| < 2^-960), so the exact
// correction x*y - p - e goes into the extended accumulator X.  If a product
// is huge (|p| >= 2^1000: the FPE's sums may have overflowed), the CTA's fast
// words are dropped and X takes all of its products exactly.  X is then added into
// gacc[XS_OFF ..].  each(f) calls f(i) for every element index i of this CTA,
// spread over its threads; X: NX * XS_L words of shared scratch (NX > 1: one
// accumulator per warp, fewer same-address atomics, summed at the end).  The
// hot loops are untouched: only flagged CTAs pay, one more read of their share.
template <int NX, class Each>
__device__ void cta_full_range(CtaSacc<1> &S, unsigned long long *X, long long *gacc, const double *x, const double *y,
                               Each each) {
    __shared__ int poisoned;
    unsigned long long *Xw = X + ((threadIdx.x >> 5) % NX) * XS_L;
    for (int i = threadIdx.x; i < NX * XS_L; i += blockDim.x) X[i] = 0ull;
    if (threadIdx.x == 0) poisoned = 0;
    __syncthreads();
    each([&](int64_t i) {
        const double a = x[i], b = y[i];
        if (!isfinite(a) || !isfinite(b)) {
            atomicOr(&S.flags, FLAG_NONFINITE);
            return;
        }
        const double p = __dmul_rn(a, b), e = __fma_rn(a, b, -p);  // as the fast pass formed them
        const unsigned ep = (unsigned)(__double2hiint(p) >> 20) & 0x7FFu;
        if (((((ep - 63u) >= 1960u) & !(is_zero(a) | is_zero(b))) | (ep == 0x7FFu)) == 0u) return;  // not flagged
        if (ep >= 63u) {  // |p| >= 2^1000: the FPE's TwoSums may have overflowed
            poisoned = 1;
            return;
        }
        xs_add_product(Xw, a, b);     // + the exact product
        xs_add_product(Xw, -p, 1.0);  // - what the FPE received
        xs_add_product(Xw, -e, 1.0);
    });
    __syncthreads();
    if (S.flags & FLAG_NONFINITE) return;
    if (poisoned) {  // the CTA's fast words are lost: all its products, exactly
        for (int i = threadIdx.x; i < NX * XS_L; i += blockDim.x) X[i] = 0ull;
        for (int i = threadIdx.x; i < SACC_L; i += blockDim.x) S.w[0][i] = 0ull;
        __syncthreads();
        each([&](int64_t i) { xs_add_product(Xw, x[i], y[i]); });
    }
    __syncthreads();
    if (NX > 1) {  // the warps' accumulators into X[0 .. XS_L) (each word < NX * 2^33 in magnitude)
        for (int i = threadIdx.x; i < XS_L; i += blockDim.x) {
            long long t = 0;
            for (int k = 0; k < NX; ++k) t += (long long)X[k * XS_L + i];
            X[i] = (unsigned long long)t;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) xs_normalize((long long *)X);
    __syncthreads();
    for (int i = threadIdx.x; i < XS_L; i += blockDim.x)
        if (X[i]) atomicAdd((unsigned long long *)&gacc[XS_OFF + i], X[i]);
}

// Whether a reduction phase uses the full-range dots (R-24): the standalone
// EXDOT always; Algorithm 2's phases (init, A, B, true residual) unless the
// solve asked for the fast zone (R-9); Algorithm 1's phases keep R-9 (R-20).
__device__ __forceinline__ bool phase_full_range(int phase, const Scalars *sc) {
    if (phase == PH_EXDOT) return true;
    if (phase >= PH1_INIT || !sc) return false;
    return sc->range_mode == 0;
}

// The exact correction of one product of finite operands a, b, as a fast
// pass formed it (p = fl(a b), e = fma(a, b, -p); a non-finite p or e was
// never deposited): X += a b - p - e.
__device__ __noinline__ void xs_correct(unsigned long long *X, double a, double b) {
    const double p = __dmul_rn(a, b), e = __fma_rn(a, b, -p);
    xs_add_product(X, a, b);
    if (isfinite(p)) {
        xs_add_product(X, -p, 1.0);
        if (isfinite(e)) xs_add_product(X, -e, 1.0);
    }
}

// Full-range pass of a CTA of an ND-dot FPE kernel whose fast pass raised
// FLAG_RANGE (R-24): all threads, after the
// CTA's FPEs are merged into S.w and before it publishes.  rows(f) calls
// f(i) for every element i of this CTA (spread over its threads);
// pair(d, i, a, b) yields dot d's operands at i, exactly as the fast pass
// formed them.  A flagged product (|fl(ab)| < 2^-960 with a, b != 0) is
// corrected into dot d's extended accumulator; a product with |fl(ab)| >=
// 2^1000 may have overflowed the FPE's sums, so that dot's fast words of this
// CTA are dropped and all its products enter the extended accumulator
// exactly.  NaN/Inf operands set FLAG_NONFINITE (the solve stops).  The
// normalised extended words are red.added into gext[d * XS_L ..].  X: ND *
// XS_L words of shared scratch.  Only flagged CTAs run this (one more read of
// their rows).
template <int ND, class Rows, class Pair>
__device__ void cta_full_range_nd(CtaSacc<ND> &S, unsigned long long *X, long long *gext, Rows rows, Pair pair) {
    __shared__ int poisoned[ND];
    for (int i = threadIdx.x; i < ND * XS_L; i += blockDim.x) X[i] = 0ull;
    if (threadIdx.x < ND) poisoned[threadIdx.x] = 0;
    __syncthreads();
    rows([&](int64_t i) {
#pragma unroll
        for (int d = 0; d < ND; ++d) {
            double a, b;
            pair(d, i, a, b);
            if (!isfinite(a) || !isfinite(b)) {
                atomicOr(&S.flags, FLAG_NONFINITE);
                continue;
            }
            if (is_zero(a) || is_zero(b)) continue;
            const double p = __dmul_rn(a, b);
            const unsigned ep = (unsigned)(__double2hiint(p) >> 20) & 0x7FFu;
            if ((ep - 63u) < 1960u) continue;  // inside the fast zone: TwoProd was exact, no correction
            if (ep >= 63u) {                   // |p| >= 2^1000 (or p = inf)
                poisoned[d] = 1;
                continue;
            }
            xs_correct(X + d * XS_L, a, b);
        }
    });
    __syncthreads();
    if (S.flags & FLAG_NONFINITE) return;
    bool any_p = false;
#pragma unroll
    for (int d = 0; d < ND; ++d) any_p |= poisoned[d] != 0;
    if (any_p) {  // the poisoned dots: every product of this CTA, exactly
        for (int j = threadIdx.x; j < ND * XS_L; j += blockDim.x)
            if (poisoned[j / XS_L]) X[j] = 0ull;
        for (int j = threadIdx.x; j < ND * SACC_L; j += blockDim.x)
            if (poisoned[j / SACC_L]) (&S.w[0][0])[j] = 0ull;
        __syncthreads();
        rows([&](int64_t i) {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                if (!poisoned[d]) continue;
                double a, b;
                pair(d, i, a, b);
                xs_add_product(X + d * XS_L, a, b);
            }
        });
        __syncthreads();
    }
    if (threadIdx.x < ND) xs_normalize((long long *)X + threadIdx.x * XS_L);
    __syncthreads();
    for (int j = threadIdx.x; j < ND * XS_L; j += blockDim.x)
        if (X[j]) atomicAdd((unsigned long long *)&gext[j], X[j]);
}

// The extended path of round_dots (kept out of line: it is rare, and inlined
// it would raise the register count of the kernels that call it): dot d =
// fast words w[d] + extended words ge[d XS_L ..], rounded once into r[d].
__device__ __noinline__ unsigned round_ext(double *r, const long long *w, long long *ge, int nd, bool nonfinite,
                                           bool clear_ext) {
    __shared__ long long X[XS_L];
    __shared__ unsigned ovf;
    __syncthreads();
    if (threadIdx.x == 0) ovf = 0u;
    for (int d = 0; d < nd; ++d) {
        long long *g = ge + d * XS_L;
        for (int i = threadIdx.x; i < XS_L; i += blockDim.x) {
            X[i] = __ldcg(&g[i]);
            if (clear_ext) g[i] = 0;
        }
        __syncthreads();
        if (threadIdx.x == 0 && !nonfinite) {
            const long long *wd = w + d * SACC_L;
            for (int i = 0; i < SACC_L; ++i) X[i + 33] += wd[i] * (1ll << 18);  // 2^-1074 = 2^(32*33+18) * 2^-2148
            xs_normalize(X);
            const double v = xs_round(X);
            r[d] = v;
            if (isinf(v)) ovf |= FLAG_RANGE;
        }
        __syncthreads();
    }
    return nonfinite ? FLAG_NONFINITE : ovf;
}

// The rounded dots of a reduction buffer whose fast words are normalised in
// S.w (cta_sacc_collect): S.rounded[0..ND), all threads.  full (R-24): when
// some CTA flagged FLAG_RANGE (and no input was NaN/Inf), dot d is its fast
// words plus its extended words gacc[xs_off(ND) + d XS_L ..], rounded once
// (RN-even, subnormals, +-inf on overflow), and those extended words are
// cleared (clear_ext; the fused kernels' CTAs all read one buffer, CTA 0
// clears it later).  Returns the flags for phase_finalize: full -> FLAG_NONFINITE,
// or FLAG_RANGE for a dot that rounds to +-inf; fast zone (R-9) -> the
// gathered flags plus overflow.
template <int ND>
__device__ unsigned round_dots(CtaSacc<ND> &S, long long *gacc, unsigned gflags, bool full, bool clear_ext = true) {
    __shared__ unsigned ovf;
    if (threadIdx.x == 0) ovf = 0u;
    __syncthreads();
    long long *w = (long long *)&S.w[0][0];
    if ((threadIdx.x >> 5) < ND) {  // one warp per dot
        bool o = false;
        const double rv = sacc_round_warp(w + (threadIdx.x >> 5) * SACC_L, &o);
        if ((threadIdx.x & 31) == 0) {
            S.rounded[threadIdx.x >> 5] = rv;
            if (o) atomicOr(&ovf, FLAG_RANGE);
        }
    }
    __syncthreads();
    if (!full) return gflags | ovf;
    if (!(gflags & FLAG_RANGE)) return (gflags & FLAG_NONFINITE) | ovf;
    return round_ext(S.rounded, (const long long *)&S.w[0][0], gacc + xs_off(ND), ND, (gflags & FLAG_NONFINITE) != 0,
                     clear_ext);
}

// Last CTA of a dot kernel: collect + normalise gacc; then either round and
// finalise (single rank) or leave normalised words for the allreduce.
template <int ND>
__device__ void last_cta_finish(CtaSacc<ND> &S, long long *gacc, unsigned *ticket, int phase, int finalize,
                                Scalars *sc, double *hist, double *out, int32_t *out_flags) {
    unsigned gflags;
    cta_sacc_collect<ND>(S, gacc, gflags);
    long long *w = (long long *)&S.w[0][0];
    if (finalize) {
        unsigned f = round_dots<ND>(S, gacc, gflags, phase_full_range(phase, sc));
        if (phase == PH_EXDOT) f |= gflags & FLAG_RANGE;  // the exdot flag contract reports the zone (pbicgstab.h)
        if (threadIdx.x == 0) phase_finalize(phase, sc, S.rounded, f, hist, out, out_flags);
        for (int i = threadIdx.x; i < ND * SACC_L + SACC_FLAGW; i += blockDim.x) gacc[i] = 0;
    } else {
        for (int i = threadIdx.x; i < ND * SACC_L; i += blockDim.x) gacc[i] = w[i];
    }
    if (threadIdx.x == 0) *ticket = 0u;
}

// ------------------------------------------------------------------------
// K2: p,s,z,q,y + phase-A partial dots
// Memory pipelining: each thread loads U row pairs (8 x 16 B each) before it
// computes any of them, so U*128 B per thread are in flight.
// ------------------------------------------------------------------------
struct K2Args {
    int64_t n;
    const double *r, *rh, *w, *t, *v;
    double *p, *s, *z, *q, *y;
    Scalars *sc;
    long long *gacc;
    unsigned *ticket;
    double *hist;
    int finalize;
    double *part;  // plain dot mode: CTA partials [grid][ND] (exact mode: unused)
    const double *minv;  // pipelined block Jacobi (R-25): M^-1 blocks of the own rows, or null
    double *zh;          // ... z_hat = M^-1 z (own part of its padded buffer)
    int last_rank;       // this rank holds the global last row (a 1x1 tail block when n is odd)
};

// ------------------------------------------------------------------------
// K3: x,r,w + phase-B partial dots
// ------------------------------------------------------------------------
struct K3Args {
    int64_t n;
    const double *rh, *p, *q, *y, *t, *v;
    double *x, *r, *w;
    Scalars *sc;
    long long *gacc;
    unsigned *ticket;
    double *hist;
    int finalize;
    double *part;  // plain dot mode: CTA partials [grid][ND] (exact mode: unused)
    const double *minv;  // pipelined block Jacobi (R-25), or null
    double *wh;          // w_hat = M^-1 w
    int last_rank;
};

// pipelined 2x2 block Jacobi (R-25): u_hat of the block (u0, u1) = rows
// (2m, 2m+1) with the formula of bj_apply_kernel / orc_bj_apply
__device__ __forceinline__ double2 bj_pair(const double *minv, int64_t m, double u0, double u1) {
    const double2 q01 = __ldg((const double2 *)minv + 2 * m), q23 = __ldg((const double2 *)minv + 2 * m + 1);
    return make_double2(__fma_rn(q01.x, u0, __dmul_rn(q01.y, u1)), __fma_rn(q23.x, u0, __dmul_rn(q23.y, u1)));
}

// ------------------------------------------------------------------------
// multidot: up to 4 fused EXDOTs (init, true residual, standalone exdot)
// ------------------------------------------------------------------------
struct MultiDotArgs {
    int64_t n;
    const double *x[4], *y[4];
    Scalars *sc;  // may be null for standalone exdot
    long long *gacc;
    unsigned *ticket;
    double *hist;
    int phase, finalize;
    double *out;
    int32_t *out_flags;
};

template <int ND, int NP, int NE, int BS, int U>
__global__ void __launch_bounds__(BS) multidot_kernel(MultiDotArgs a) {
    __shared__ CtaSacc<ND> S;
    if (a.sc && a.sc->done && a.phase != PH_TRUE) return;
    cta_sacc_zero<ND>(S);
    __syncthreads();
    ExAcc<NP, NE> acc[ND];
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d].zero();
    unsigned flags = 0;
    const int64_t n = a.n;
    const int64_t stride = (int64_t)gridDim.x * BS;
    const int64_t k = (int64_t)blockIdx.x * BS + threadIdx.x;
    bool aligned = true;
#pragma unroll
    for (int d = 0; d < ND; ++d) aligned &= ((((uintptr_t)a.x[d]) | ((uintptr_t)a.y[d])) & 15) == 0;
    if (aligned) {
        const int64_t npair = n >> 1;
        const int64_t full = (npair / (stride * U)) * (stride * U);
        for (int64_t base = k; base < full; base += stride * U) {
            double2 xv[U][ND], yv[U][ND];
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int d = 0; d < ND; ++d) {
                    xv[u][d] = __ldcs((const double2 *)a.x[d] + base + u * stride);
                    yv[u][d] = __ldcs((const double2 *)a.y[d] + base + u * stride);
                }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int d = 0; d < ND; ++d) {
                    acc[d].template add<true>(xv[u][d].x, yv[u][d].x, S.w[d], flags);
                    acc[d].template add<true>(xv[u][d].y, yv[u][d].y, S.w[d], flags);
                }
        }
        for (int64_t i = full + k; i < npair; i += stride) {
#pragma unroll
            for (int d = 0; d < ND; ++d) {
                const double2 xv = ((const double2 *)a.x[d])[i], yv = ((const double2 *)a.y[d])[i];
                acc[d].template add<false>(xv.x, yv.x, S.w[d], flags);
                acc[d].template add<false>(xv.y, yv.y, S.w[d], flags);
            }
        }
        if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
#pragma unroll
            for (int d = 0; d < ND; ++d) acc[d].template add<false>(a.x[d][n - 1], a.y[d][n - 1], S.w[d], flags);
        }
    } else {
        for (int64_t i = k; i < n; i += stride) {
#pragma unroll
            for (int d = 0; d < ND; ++d) acc[d].template add<false>(a.x[d][i], a.y[d][i], S.w[d], flags);
        }
    }
#pragma unroll
    for (int d = 0; d < ND; ++d) acc[d].warp_merge(S.w[d]);
    // full range (R-24): the CTAs that met a product outside the fast zone
    // correct it (the standalone EXDOT, single GPU or distributed; Alg. 2's
    // init and true-residual dots unless the solve runs in the fast zone)
    if (a.phase == PH_EXDOT || phase_full_range(a.phase, a.sc)) {
        if (flags) atomicOr(&S.flags, flags);
        flags = 0;
        __syncthreads();
        auto rows = [&](auto f) {  // this CTA's elements, as the fast pass visited them
            const bool al = aligned;
            const int64_t m = al ? n >> 1 : n;  // pairs (aligned) or elements
            for (int64_t p0 = (int64_t)blockIdx.x * BS; p0 < m; p0 += stride)
                for (int64_t p = p0 + threadIdx.x; p < min(p0 + BS, m); p += blockDim.x) {
                    if (al) { f(2 * p); f(2 * p + 1); } else f(p);
                }
            if (al && (n & 1) && blockIdx.x == 0 && threadIdx.x == 0) f(n - 1);
        };
        if constexpr (ND == 1) {
            if (a.phase == PH_EXDOT) {
                __shared__ unsigned long long X1[XS_L];
                if (S.flags) cta_full_range<1>(S, X1, a.gacc, a.x[0], a.y[0], rows);
            }
        }
        if (a.phase != PH_EXDOT && (S.flags & FLAG_RANGE)) {
            __shared__ unsigned long long X[ND * XS_L];
            cta_full_range_nd<ND>(S, X, a.gacc + xs_off(ND), rows, [&](int d, int64_t i, double &x, double &y) {
                x = a.x[d][i];
                y = a.y[d][i];
            });
        }
    }
    if (cta_sacc_publish<ND>(S, flags, a.gacc, a.ticket))
        last_cta_finish<ND>(S, a.gacc, a.ticket, a.phase, a.finalize, a.sc, a.hist, a.out, a.out_flags);
}

// After an allreduce of normalised words: normalise, round, finalise (1 CTA).
template <int ND>
__global__ void finalize_kernel(long long *gacc, int phase, Scalars *sc, double *hist, double *out,
                                int32_t *out_flags) {
    __shared__ CtaSacc<ND> S;
    if (sc && sc->done && phase != PH_TRUE && phase != PH_EXDOT) {
        for (int i = threadIdx.x; i < ND * SACC_L + SACC_FLAGW; i += blockDim.x) gacc[i] = 0;
        return;
    }
    if (threadIdx.x == 0) S.flags = 0u;
    unsigned gflags;
    cta_sacc_collect<ND>(S, gacc, gflags);
    unsigned f = round_dots<ND>(S, gacc, gflags, phase_full_range(phase, sc));
    if (phase == PH_EXDOT) f |= gflags & FLAG_RANGE;  // the exdot flag contract reports the zone (pbicgstab.h)
    if (threadIdx.x == 0) phase_finalize(phase, sc, S.rounded, f, hist, out, out_flags);
    __syncthreads();
    for (int i = threadIdx.x; i < ND * SACC_L + SACC_FLAGW; i += blockDim.x) gacc[i] = 0;
}

// Virtual-rank "allreduce": every rank's gacc := sum over ranks (int64).
__global__ void vallreduce_kernel(long long **gaccs, int nr, int words) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += gridDim.x * blockDim.x) {
        long long s = 0;
        for (int r = 0; r < nr; ++r) s += gaccs[r][i];
        for (int r = 0; r < nr; ++r) gaccs[r][i] = s;
    }
}

// ------------------------------------------------------------------------
// SpMV on sliced ELL (C = 32 rows per slice, slot-major), one thread per row.
// The per-row chain is left to right in ascending column order starting from
// +0.0, one fma per nonzero; padding slots are never folded (R-6).
// ------------------------------------------------------------------------
struct SellMat {
    int64_t n;
    const int64_t *slice_off;  // nslices+1, element offsets of each slice
    const int32_t *row_len;    // by position
    const double *val;
    const int32_t *col;        // x-buffer index of the nonzero minus the position (pos-relative)
    const int32_t *perm;       // position -> row (sigma-sorted windows), or null (identity)
    // Per slice-slot column offsets (index compression of the sliced ELL):
    // SELL_RS int32 per slice s: rec[16 s + 15] = mask; bit k (k < 15) set
    // <=> every row of slice s that has a k-th nonzero finds it at x-buffer
    // index pos + rec[16 s + k]; the column ids of that slice-slot are then
    // never read.  Slots k >= 15 are always explicit.  Null: every slot
    // explicit.  The same nonzeros are folded in the same order (R-6).
    const int32_t *slot_rec;
    // positions [p0, p1) this launch folds (interior / boundary split of a
    // rank's rows under multi-rank halo overlap; default: all rows)
    int64_t p0, p1;
};

static constexpr int SELL_RS = 16, SELL_MASK = 15;

static constexpr int32_t SELL_EXPLICIT = INT32_MIN;

enum { SPMV_PLAIN = 0, SPMV_RESID = 1 };

template <int MODE, int UNR, int RPT>
__global__ void __launch_bounds__(256) spmv_sell_kernel(SellMat A, const double *__restrict__ x,
                                                        double *__restrict__ y, const double *__restrict__ b,
                                                        double *__restrict__ y2, const Scalars *sc) {
    // RPT positions per thread (pos0 + 256*u), loads of all of them in flight
    // before any fold: more memory-level parallelism per thread.
    pdl_wait();
    if (sc && sc->done) return;
    const int64_t pos0 = A.p0 + (int64_t)blockIdx.x * (256 * RPT) + threadIdx.x;
    int64_t base[RPT];
    int len[RPT], lmax = 0;
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t pos = pos0 + 256 * u;
        base[u] = 0;
        len[u] = 0;
        if (pos < A.p1) {
            base[u] = __ldg(&A.slice_off[pos >> 5]) + (pos & 31);
            len[u] = __ldg(&A.row_len[pos]);
        }
        lmax = max(lmax, len[u]);
    }
    double acc[RPT];
#pragma unroll
    for (int u = 0; u < RPT; ++u) acc[u] = 0.0;
    for (int k = 0; k < lmax; k += UNR) {
        double v[RPT][UNR], xv[RPT][UNR];
        int c[RPT][UNR];
#pragma unroll
        for (int u = 0; u < RPT; ++u)
#pragma unroll
            for (int j = 0; j < UNR; ++j)
                if (k + j < len[u]) {
                    v[u][j] = __ldcs(A.val + base[u] + 32 * (k + j));
                    c[u][j] = __ldcs(A.col + base[u] + 32 * (k + j));
                }
#pragma unroll
        for (int u = 0; u < RPT; ++u)
#pragma unroll
            for (int j = 0; j < UNR; ++j)
#ifdef PBCG_EXP_NOGATHER  // timing experiment only (wrong results): coalesced x reads
                if (k + j < len[u]) xv[u][j] = __ldg(x + (pos0 + 256 * u + (c[u][j] & 1)));
#else
                if (k + j < len[u]) xv[u][j] = __ldg(x + (pos0 + 256 * u + c[u][j]));
#endif
#pragma unroll
        for (int u = 0; u < RPT; ++u)
#pragma unroll
            for (int j = 0; j < UNR; ++j)
                if (k + j < len[u]) acc[u] = __fma_rn(v[u][j], xv[u][j], acc[u]);
    }
#pragma unroll
    for (int u = 0; u < RPT; ++u) {
        const int64_t pos = pos0 + 256 * u;
        if (pos >= A.p1) continue;
        const int64_t row = A.perm ? (int64_t)__ldg(&A.perm[pos]) : pos;
        if (MODE == SPMV_PLAIN) {
            y[row] = acc[u];
        } else {
            const double r = __dsub_rn(b[row], acc[u]);  // r0 := b - A x0 (l.64), one rounding
            y[row] = r;
            if (y2) y2[row] = r;
        }
    }
}

// Software-pipelined SELL SpMV.  A thread owns positions pos, pos + stride,
// ... (persistent grid).  Work is a stream of batches of UNR slots: while the
// x-gathers of batch j are in flight, the val/col loads of batch j+1 (the next
// batch of this row, or the first batch of the next row, whose descriptor was
// loaded one row ahead) are already issued.  Each thread therefore waits on
// one round trip per batch instead of three per row (descriptor -> val/col ->
// x).  The fold is unchanged: one fma per nonzero, ascending columns, +0.0
// start, never over padding (R-6).
template <int MODE, int UNR>
__global__ void __launch_bounds__(256) spmv_sell_pipe_kernel(SellMat A, const double *__restrict__ x,
                                                             double *__restrict__ y, const double *__restrict__ b,
                                                             double *__restrict__ y2, const Scalars *sc) {
    pdl_sync();
    if (sc && sc->done) return;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    int64_t pos = A.p0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // descriptor of a position: slot-0 offset and row length (0 past the end)
    auto desc = [&](int64_t p, int64_t &base, int &len) {
        base = 0;
        len = 0;
        if (p < A.p1) {
            base = __ldg(&A.slice_off[p >> 5]) + (p & 31);
            len = __ldg(&A.row_len[p]);
        }
    };
    auto load_vc = [&](int64_t base, int k0, int len, double *v, int *c) {
#pragma unroll
        for (int j = 0; j < UNR; ++j)
            if (k0 + j < len) {
                v[j] = __ldcs(A.val + base + 32 * (k0 + j));
                c[j] = __ldcs(A.col + base + 32 * (k0 + j));
            }
    };
    int64_t cbase, nbase;
    int clen, nlen;
    desc(pos, cbase, clen);
    desc(pos + stride, nbase, nlen);
    double v[UNR], vn[UNR], xv[UNR];
    int c[UNR], cn[UNR];
    load_vc(cbase, 0, clen, v, c);
    while (pos < A.p1) {
        double acc = 0.0;
        for (int k0 = 0;; k0 += UNR) {
#pragma unroll
            for (int j = 0; j < UNR; ++j)
                if (k0 + j < clen) xv[j] = __ldg(x + (pos + c[j]));
            const bool more = k0 + UNR < clen;
            // prefetch the next batch: rest of this row, or the next row's first
            int64_t nnbase = 0;
            int nnlen = 0;
            if (more) {
                load_vc(cbase, k0 + UNR, clen, vn, cn);
            } else {
                load_vc(nbase, 0, nlen, vn, cn);
                desc(pos + 2 * stride, nnbase, nnlen);
            }
#pragma unroll
            for (int j = 0; j < UNR; ++j)
                if (k0 + j < clen) acc = __fma_rn(v[j], xv[j], acc);
#pragma unroll
            for (int j = 0; j < UNR; ++j) {
                v[j] = vn[j];
                c[j] = cn[j];
            }
            if (!more) {
                const int64_t row = A.perm ? (int64_t)__ldg(&A.perm[pos]) : pos;
                if (MODE == SPMV_PLAIN) {
                    y[row] = acc;
                } else {
                    const double r = __dsub_rn(b[row], acc);  // r0 := b - A x0 (l.64)
                    y[row] = r;
                    if (y2) y2[row] = r;
                }
                pos += stride;
                cbase = nbase;
                clen = nlen;
                nbase = nnbase;
                nlen = nnlen;
                break;
            }
        }
    }
}

// ------------------------------------------------------------------------
// Algorithm 1 vector updates, the oracle's arithmetic
// (orc_bicgstab_dots): separate RN multiply / add, left to right, no fma.
// ------------------------------------------------------------------------
__global__ void a1_q_kernel(int64_t n, const double *r, const double *s, double *q, const Scalars *sc) {
    if (sc->done) return;
    const double a = sc->alpha;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        q[k] = __dsub_rn(r[k], __dmul_rn(a, s[k]));  // q := r - a s
}

__global__ void a1_xconv_kernel(int64_t n, double *x, const double *p, const Scalars *sc) {
    if (!sc->qconv) return;
    const double a = sc->alpha;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        x[k] = __dadd_rn(x[k], __dmul_rn(a, p[k]));  // x := x + a p (converged at the q check)
}

__global__ void a1_qclear_kernel(Scalars *sc) { sc->qconv = 0; }

__global__ void a1_xr_kernel(int64_t n, double *x, const double *p, const double *q, const double *y, double *r,
                             const Scalars *sc) {
    if (sc->done) return;
    const double a = sc->alpha, om = sc->omega;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
        const double qk = q[k];
        x[k] = __dadd_rn(__dadd_rn(x[k], __dmul_rn(a, p[k])), __dmul_rn(om, qk));  // x := x + a p + w q
        r[k] = __dsub_rn(qk, __dmul_rn(om, y[k]));                                 // r := q - w y
    }
}

__global__ void a1_p_kernel(int64_t n, const double *r, double *p, const double *s, const Scalars *sc) {
    if (sc->done) return;
    const double be = sc->beta, om = sc->omega;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x)
        p[k] = __dadd_rn(r[k], __dmul_rn(be, __dsub_rn(p[k], __dmul_rn(om, s[k]))));  // p := r + b (p - w s)
}

// Plain dot mode: d[k] = sum over ranks v (in order) and CTAs c (in order) of
// part[v][c*ND + k], then the phase's scalar step (the same phase_finalize as
// the exact mode).  pd (if not null) receives d[] (NCCL ranks: the local sums,
// allreduced before plain_phase_kernel).
template <int ND>
__global__ void plain_finalize_kernel(const double *const *parts, int V, int grid, int phase, Scalars *sc,
                                      double *hist, double *pd, int run_phase) {
    __shared__ double d[ND];
    if (threadIdx.x < ND) {
        double t = 0.0;
        for (int v = 0; v < V; ++v)
            for (int c = 0; c < grid; ++c) t = __dadd_rn(t, parts[v][(size_t)c * ND + threadIdx.x]);
        d[threadIdx.x] = t;
        if (pd) pd[threadIdx.x] = t;
    }
    __syncthreads();
    if (run_phase && threadIdx.x == 0) phase_finalize(phase, sc, d, 0u, hist, nullptr, nullptr);
}

__global__ void plain_phase_kernel(int phase, Scalars *sc, const double *pd, double *hist) {
    if (threadIdx.x == 0) phase_finalize(phase, sc, pd, 0u, hist, nullptr, nullptr);
}

// ------------------------------------------------------------------------
// setup helpers
// ------------------------------------------------------------------------
// column hull of rows [r0,r1): out[0] = min col, out[1] = max col (unchanged if no nonzeros)
__global__ void row_hull_kernel(int64_t r0, int64_t r1, const int32_t *rp, const int32_t *col, long long *out) {
    int lo = INT32_MAX, hi = INT32_MIN;
    for (int64_t r = r0 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < r1; r += (int64_t)gridDim.x * blockDim.x) {
        const int32_t s = rp[r], e = rp[r + 1];
        if (e > s) {
            lo = min(lo, col[s]);
            hi = max(hi, col[e - 1]);
        }
    }
    lo = __reduce_min_sync(0xFFFFFFFFu, lo);
    hi = __reduce_max_sync(0xFFFFFFFFu, hi);
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(&out[0], (long long)lo);
        atomicMax(&out[1], (long long)hi);
    }
}

// CSR rows -> sliced ELL.  rp is indexed by local row and holds absolute
// offsets into col/val.  Checks: finite values, strictly increasing columns in
// [0, ncols), row pointer monotone.
__global__ void csr_to_sell_kernel(int64_t n, const int32_t *rp, const int32_t *col, const double *val,
                                   int64_t ncols, int64_t col_shift, const int64_t *slice_off, int32_t *row_len,
                                   double *sval, int32_t *scol, const int32_t *perm, int *bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t src = perm ? perm[r] : r;  // r is the SELL position
        const int32_t s = rp[src], e = rp[src + 1];
        const int len = e - s;
        if (len < 0) { atomicOr(bad, 1); continue; }
        row_len[r] = len;
        const int64_t base = slice_off[r >> 5] + (r & 31);
        int32_t prev = -1;
        for (int k = 0; k < len; ++k) {
            const int32_t c = col[s + k];
            const double v = val[s + k];
            if (c <= prev || c < 0 || (int64_t)c >= ncols) atomicOr(bad, 1);
            if (!isfinite(v)) atomicOr(bad, 2);
            prev = c;
            sval[base + 32 * k] = v;
            scol[base + 32 * k] = (int32_t)((int64_t)c - col_shift - r);  // pos-relative
        }
        const int64_t width = (slice_off[(r >> 5) + 1] - slice_off[r >> 5]) >> 5;
        for (int64_t k = len; k < width; ++k) {  // padding: never folded, kept addressable
            sval[base + 32 * k] = 0.0;
            scol[base + 32 * k] = 0;
        }
    }
}

// Slot records of the sliced ELL (SellMat::slot_rec): one warp per slice.
// For slot k < SELL_MASK the lanes whose row has a k-th nonzero compare their
// pos-relative column; all equal -> record it and set mask bit k.  n_explicit
// counts the column ids that stay explicit (the format's index bytes).
__global__ void sell_slot_records_kernel(int64_t n, int64_t nslices, const int64_t *slice_off, const int32_t *row_len,
                                         const int32_t *scol, int32_t *slot_rec, unsigned long long *n_explicit) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    unsigned long long expl = 0;
    for (int64_t sl = wid; sl < nslices; sl += nw) {
        const int64_t pos = sl * 32 + lane;
        const int len = pos < n ? row_len[pos] : 0;
        const int64_t so = slice_off[sl];
        const int64_t width = (slice_off[sl + 1] - so) >> 5;
        uint32_t mask = 0;
        int32_t d_lane = 0;  // lane k keeps the record of slot k
        for (int64_t k = 0; k < width; ++k) {
            const bool act = k < len;
            const int d = act ? scol[so + lane + 32 * k] : 0;
            const int dmin = __reduce_min_sync(0xFFFFFFFFu, act ? d : INT32_MAX);
            const int dmax = __reduce_max_sync(0xFFFFFFFFu, act ? d : INT32_MIN);
            const unsigned m = __ballot_sync(0xFFFFFFFFu, act);
            const bool uni = dmin == dmax && k < SELL_MASK;
            if (uni) {
                mask |= 1u << k;
                if (lane == k) d_lane = dmin;
            } else {
                expl += __popc(m);
            }
        }
        if (lane < SELL_RS) slot_rec[sl * SELL_RS + lane] = lane == SELL_MASK ? (int32_t)mask : d_lane;
    }
    if (lane == 0 && expl) atomicAdd(n_explicit, expl);
}

// Right Jacobi preconditioning (NEXT-3, R-22).  d[r] := A(row0 + r, row0 + r)
// (the stored diagonal; missing or zero -> bad |= 4).
__global__ void diag_kernel(int64_t n, int64_t row0, const int32_t *rp, const int32_t *col, const double *val,
                            double *d, int *bad) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (int64_t)gridDim.x * blockDim.x) {
        double v = 0.0;
        for (int32_t k = rp[r]; k < rp[r + 1]; ++k)
            if ((int64_t)col[k] == row0 + r) v = val[k];
        d[r] = v;
        if (v == 0.0) atomicOr(bad, 4);
    }
}

// A' = A D^-1 on the sliced ELL: every stored entry divided (RN) by the
// diagonal of its column, read from the padded x-layout copy of d (halo incl.)
__global__ void sell_colscale_kernel(int64_t n, const int64_t *slice_off, const int32_t *row_len, double *sval,
                                     const int32_t *scol, const double *dpad) {
    for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < n;
         pos += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = slice_off[pos >> 5] + (pos & 31);
        const int len = row_len[pos];
        for (int k = 0; k < len; ++k)
            sval[base + 32 * k] = __ddiv_rn(sval[base + 32 * k], dpad[pos + scol[base + 32 * k]]);
    }
}

// ------------------------------------------------------------------------
// 2x2 point-block Jacobi, right preconditioning (SURVEY §8(f) NEXT-3,
// DESIGN.md R-23): M = the 2x2 diagonal blocks of A (global rows 2m, 2m+1; a
// 1x1 block for the last row when n is odd), B = A M^-1 stored explicitly.
// B's pattern: every block a row touches contributes both its columns.
// Per block (a b; c d): det = fma(a, d, -(b c)), M^-1 = (d -b; -c a) / det
// (one RN division each); B_i,2m = fma(A_i,2m, m00, A_i,2m+1 m10),
// B_i,2m+1 = fma(A_i,2m, m01, A_i,2m+1 m11); y = M x and x = M^-1 y per
// block with the same shape of formula.
// ------------------------------------------------------------------------
// entries of row r of B: 2 per distinct column block (1 for the odd tail)
__global__ void bj_count_kernel(int64_t nloc, const int32_t *rp, const int32_t *col, int64_t n, int32_t *cnt) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nloc; r += (int64_t)gridDim.x * blockDim.x) {
        int c = 0;
        int64_t last = -1;
        for (int32_t k = rp[r]; k < rp[r + 1]; ++k) {
            const int64_t m = col[k] >> 1;
            if (m != last) c += (2 * m + 1 < n) ? 2 : 1;
            last = m;
        }
        cnt[r] = c;
    }
}

// B's pattern, with A's values at A's columns and +0.0 at the added ones
__global__ void bj_fill_kernel(int64_t nloc, const int32_t *rp, const int32_t *col, const double *val, int64_t n,
                               const int32_t *brp, int32_t *bcol, double *bval) {
    for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < nloc; r += (int64_t)gridDim.x * blockDim.x) {
        int32_t o = brp[r];
        for (int32_t k = rp[r]; k < rp[r + 1];) {
            const int64_t m = col[k] >> 1;
            double v0 = 0.0, v1 = 0.0;
            for (; k < rp[r + 1] && (col[k] >> 1) == m; ++k) {
                if (col[k] & 1) v1 = val[k];
                else v0 = val[k];
            }
            bcol[o] = (int32_t)(2 * m);
            bval[o++] = v0;
            if (2 * m + 1 < n) {
                bcol[o] = (int32_t)(2 * m + 1);
                bval[o++] = v1;
            }
        }
    }
}

// value of A at (row r, global column c): 0 if not stored
__device__ __forceinline__ double csr_at(const int32_t *rp, const int32_t *col, const double *val, int64_t r,
                                         int64_t c) {
    for (int32_t k = rp[r]; k < rp[r + 1]; ++k)
        if (col[k] == c) return val[k];
    return 0.0;
}

// per own block (rows rb+2j, rb+2j+1; rb even): M and M^-1 (4 doubles each,
// row-major; the 1x1 tail block keeps one), and the columns of M^-1 in the
// padded x layout: c0[k] = M^-1[2m][k], c1[k] = M^-1[2m+1][k] for k in block m
__global__ void bj_blocks_kernel(int64_t nloc, int64_t rb, int64_t n, const int32_t *rp, const int32_t *col,
                                 const double *val, double *bm, double *bi, double *c0, double *c1, int *bad) {
    const int64_t nb = (nloc + 1) / 2;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r0 = 2 * j, g0 = rb + r0;
        if (g0 + 1 < n) {
            const double a = csr_at(rp, col, val, r0, g0), b = csr_at(rp, col, val, r0, g0 + 1);
            const double c = csr_at(rp, col, val, r0 + 1, g0), d = csr_at(rp, col, val, r0 + 1, g0 + 1);
            const double det = __fma_rn(a, d, -__dmul_rn(b, c));
            const double m00 = __ddiv_rn(d, det), m01 = -__ddiv_rn(b, det), m10 = -__ddiv_rn(c, det),
                         m11 = __ddiv_rn(a, det);
            if (!(det != 0.0) || !isfinite(m00) || !isfinite(m01) || !isfinite(m10) || !isfinite(m11)) atomicOr(bad, 4);
            bm[4 * j] = a; bm[4 * j + 1] = b; bm[4 * j + 2] = c; bm[4 * j + 3] = d;
            bi[4 * j] = m00; bi[4 * j + 1] = m01; bi[4 * j + 2] = m10; bi[4 * j + 3] = m11;
            c0[r0] = m00; c1[r0] = m10;
            c0[r0 + 1] = m01; c1[r0 + 1] = m11;
        } else {  // 1x1 tail block
            const double a = csr_at(rp, col, val, r0, g0);
            const double m = __ddiv_rn(1.0, a);
            if (!(a != 0.0) || !isfinite(m)) atomicOr(bad, 4);
            bm[4 * j] = a; bm[4 * j + 1] = 0.0; bm[4 * j + 2] = 0.0; bm[4 * j + 3] = 0.0;
            bi[4 * j] = m; bi[4 * j + 1] = 0.0; bi[4 * j + 2] = 0.0; bi[4 * j + 3] = 0.0;
            c0[r0] = m; c1[r0] = 0.0;
        }
    }
}

// B = A M^-1 in place on the sliced ELL of B's pattern (both columns of a
// block sit in consecutive slots): c0/c1 in the padded x layout (halo incl.),
// g = x-buffer index + buf_lo is the global column
__global__ void bj_values_kernel(int64_t nloc, int64_t n, int64_t buf_lo, const int64_t *slice_off,
                                 const int32_t *row_len, double *sval, const int32_t *scol, const double *c0,
                                 const double *c1) {
    for (int64_t pos = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; pos < nloc;
         pos += (int64_t)gridDim.x * blockDim.x) {
        const int64_t base = slice_off[pos >> 5] + (pos & 31);
        const int len = row_len[pos];
        for (int k = 0; k < len;) {
            const int64_t xi = pos + scol[base + 32 * k], g = xi + buf_lo;
            if (g + 1 < n) {  // a 2x2 block: slots k (column 2m) and k+1 (column 2m+1)
                const double v0 = sval[base + 32 * k], v1 = sval[base + 32 * (k + 1)];
                sval[base + 32 * k] = __fma_rn(v0, c0[xi], __dmul_rn(v1, c1[xi]));
                sval[base + 32 * (k + 1)] = __fma_rn(v0, c0[xi + 1], __dmul_rn(v1, c1[xi + 1]));
                k += 2;
            } else {  // the 1x1 tail block
                sval[base + 32 * k] = __dmul_rn(sval[base + 32 * k], c0[xi]);
                k += 1;
            }
        }
    }
}

// y = Q x per own block (Q = M or M^-1, 4 doubles per block), in place allowed
__global__ void bj_apply_kernel(int64_t nloc, int64_t rb, int64_t n, const double *q, const double *x, double *y) {
    const int64_t nb = (nloc + 1) / 2;
    for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nb; j += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r0 = 2 * j;
        if (rb + r0 + 1 < n) {
            const double x0 = x[r0], x1 = x[r0 + 1];
            y[r0] = __fma_rn(q[4 * j], x0, __dmul_rn(q[4 * j + 1], x1));
            y[r0 + 1] = __fma_rn(q[4 * j + 2], x0, __dmul_rn(q[4 * j + 3], x1));
        } else {
            y[r0] = __dmul_rn(q[4 * j], x[r0]);
        }
    }
}

// y := a op b elementwise (op 0: multiply, 1: divide), RN
__global__ void vec_muldiv_kernel(int64_t n, const double *a, const double *b, double *y, int op) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        y[i] = op ? __ddiv_rn(a[i], b[i]) : __dmul_rn(a[i], b[i]);
}

// Multi-rank halo overlap: flag[s] = 1 if some stored entry of slice s reads
// an x-buffer entry outside this rank's own rows [own_lo, own_hi) (a halo
// entry), so the slice must wait for the exchange; one warp per slice.
__global__ void sell_halo_flags_kernel(int64_t n, int64_t nslices, const int64_t *slice_off, const int32_t *row_len,
                                       const int32_t *scol, int64_t own_lo, int64_t own_hi, uint8_t *flag) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < nslices; sl += nw) {
        const int64_t pos = sl * 32 + lane;
        const int len = pos < n ? row_len[pos] : 0;
        const int64_t so = slice_off[sl];
        bool out = false;
        for (int k = 0; k < len; ++k) {
            const int64_t c = pos + scol[so + 32 * k + lane];  // pos-relative column
            out |= (c < own_lo) | (c >= own_hi);
        }
        const unsigned any = __ballot_sync(0xFFFFFFFFu, out);
        if (lane == 0) flag[sl] = any ? 1 : 0;
    }
}

// per slice: the largest x-buffer index its rows read (-1: no nonzero)
__global__ void sell_xmax_kernel(int64_t n, int64_t nslices, const int64_t *slice_off, const int32_t *row_len,
                                 const int32_t *scol, int64_t *xmax) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t sl = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; sl < nslices; sl += nw) {
        const int64_t pos = sl * 32 + lane;
        const int len = pos < n ? row_len[pos] : 0;
        const int64_t so = slice_off[sl];
        long long m = -1;
        for (int k = 0; k < len; ++k) m = max(m, (long long)(pos + scol[so + 32 * k + lane]));
#pragma unroll
        for (int o = 16; o; o >>= 1) m = max(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (lane == 0) xmax[sl] = m;
    }
}

// pbcg_result.digest: FNV-1a 64 over the per-row FNV-1a 64 hashes of history
// rows [0, rows) (12 doubles each, bit patterns as 64-bit words).  One warp:
// the lanes hash rows, lane 0 folds the row hashes in order.
__global__ void hist_digest_kernel(const double *hist, Scalars *sc) {
    constexpr unsigned long long B = 0xcbf29ce484222325ull, P = 0x100000001b3ull;
    const int rows = min(sc->it + 1, sc->hist_cap);
    const int lane = threadIdx.x & 31;
    unsigned long long h = B;
    for (int r0 = 0; r0 < rows; r0 += 32) {
        const int r = r0 + lane;
        unsigned long long rh = B;
        if (r < rows)
            for (int c = 0; c < H_COLS; ++c) rh = (rh ^ (unsigned long long)__double_as_longlong(hist[(size_t)r * H_COLS + c])) * P;
        for (int k = 0; k < 32 && r0 + k < rows; ++k) {
            const unsigned long long v = __shfl_sync(0xFFFFFFFFu, rh, k);
            h = (h ^ v) * P;
        }
    }
    if (lane == 0) sc->digest = h;
}

__global__ void nonfinite_scan_kernel(int64_t n, const double *v, int *bad) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        if (!isfinite(v[i])) atomicOr(bad, 2);
}

// ------------------------------------------------------------------------
// plain fp64 dot (measurement baseline, BASELINE.json north_star): grid-stride
// + warp shuffle tree + CTA partials, last CTA sums the partials in order.
// ------------------------------------------------------------------------
template <int BS>
__global__ void __launch_bounds__(BS) plain_dot_kernel(int64_t n, const double *x, const double *y,
                                                        double *partials, unsigned *ticket, double *out) {
    __shared__ double red[BS / 32];
    __shared__ int last;
    double s = 0.0;
    const int64_t npair = n >> 1;
    const int64_t stride = (int64_t)gridDim.x * BS;
    int64_t k = (int64_t)blockIdx.x * BS + threadIdx.x;
    // 4 independent pairs in flight per thread, then the remainder
    double s4[4] = {0.0, 0.0, 0.0, 0.0};
    for (; k + 3 * stride < npair; k += 4 * stride) {
        double2 a[4], b[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            a[u] = __ldcs((const double2 *)x + k + u * stride);
            b[u] = __ldcs((const double2 *)y + k + u * stride);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) s4[u] = __fma_rn(a[u].y, b[u].y, __fma_rn(a[u].x, b[u].x, s4[u]));
    }
    for (; k < npair; k += stride) {
        const double2 a = ((const double2 *)x)[k], b = ((const double2 *)y)[k];
        s = __fma_rn(a.x, b.x, s);
        s = __fma_rn(a.y, b.y, s);
    }
    s = __dadd_rn(__dadd_rn(s, s4[0]), __dadd_rn(__dadd_rn(s4[1], s4[2]), s4[3]));
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) s = __fma_rn(x[n - 1], y[n - 1], s);
    for (int o = 16; o; o >>= 1) s = __dadd_rn(s, __shfl_down_sync(0xFFFFFFFFu, s, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int i = 0; i < BS / 32; ++i) t = __dadd_rn(t, red[i]);
        partials[blockIdx.x] = t;
        __threadfence();
        last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    }
    __syncthreads();
    if (last && threadIdx.x == 0) {
        __threadfence();
        double t = 0.0;
        for (unsigned i = 0; i < gridDim.x; ++i) t = __dadd_rn(t, __ldcg(&partials[i]));
        *out = t;
        *ticket = 0u;
    }
}

}  // namespace pbcg
