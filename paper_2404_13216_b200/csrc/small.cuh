// small.cuh -- the whole p-BiCGStab iteration (Alg. 2 l.70-82) in ONE
// persistent kernel, for systems small enough that the six-kernel iteration
// is launch- and dependency-latency bound (C1: 4,096 rows).
//
// B200 design (DESIGN.md §5 "Fused small-system kernel"): a cooperative grid
// of G CTAs (co-residency guaranteed by the cooperative launch), each owning
// a contiguous range of 256-row sigma windows -- so the rows its K2/K3 part
// updates are exactly the rows its SpMV part produces, and v, t never cross
// CTAs (rows not permuted: whole 32-row slices, so up to one CTA per slice).
// Per iteration:
//   K2 rows + phase-A products (each lane deposits its own p and e: one or
//     two rows per lane, no warp aggregation) -> CTA superaccumulator ->
//     int64 red into gA
//   grid barrier (z of every row and every CTA's words are complete)
//   every CTA: normalise + round the 4 dots, the scalar step (omega) on its
//     own copy of the scalars (CTA 0: the global ones + the history)
//   SpMV v = A z over its rows; CTA barrier
//   K3 rows + phase-B products -> gB; grid barrier; round, beta/alpha'/stop
//   SpMV t = A w over its rows; CTA barrier
// Two grid barriers per iteration instead of six launches and two
// fork/joins.  The arithmetic is the same as the six-kernel path element by
// element (FMA policy F, the per-row fma chain of the SpMV, exact dots), so
// the trajectory is bit-identical to it and to the oracle.
#pragma once
#include "kernels.cuh"

namespace pbcg {

// Debug build (-DPBCG_DEBUG_COUNTERS): CTA 0 adds the globaltimer time of
// each phase to g_dbg slots (tools/diag_small.py)
#ifdef PBCG_DEBUG_COUNTERS
#define SMALL_TS(slot)                                                                 \
    do {                                                                               \
        if (blockIdx.x == 0 && threadIdx.x == 0) {                                     \
            unsigned long long t_;                                                     \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
            if ((slot) >= 0) g_dbg[(slot)] += t_ - ts_prev;                            \
            ts_prev = t_;                                                              \
        }                                                                              \
    } while (0)
#else
#define SMALL_TS(slot) ((void)0)
#endif

struct SmallArgs {
    int64_t n;
    const int64_t *slice_off;
    const int32_t *row_len;
    const double *val;
    const int32_t *col;   // pos-relative x-buffer index
    const int32_t *perm;  // position -> row, or null
    double *x, *r, *rh, *p, *s, *q, *y, *t, *v;
    double *z, *w;               // own rows of the padded buffers
    const double *zpad, *wpad;   // padded bases (x-buffer index 0)
    long long *gA[2], *gB[2];    // phase buffers, by iteration parity
    unsigned *bar;               // grid barrier: [0] arrivals, [1] generation
    Scalars *sc;
    double *hist;
    int iters;                   // at most this many iterations in this launch
};

// Sense-by-generation grid barrier (all CTAs co-resident: cooperative launch).
__device__ __forceinline__ void grid_barrier(unsigned *bar) {
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile unsigned *gen = bar + 1;
        const unsigned g0 = *gen;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            atomicExch(bar, 0u);
            __threadfence();
            atomicAdd(bar + 1, 1u);
        } else {
            while (*gen == g0) __nanosleep(20);
        }
        __threadfence();
    }
    __syncthreads();
}

// this CTA's words into the phase buffer, not normalised: the whole grid adds
// at most 2 n <= 2^18 signed 32-bit digits into any word (< 2^51, no int64
// overflow); the readers normalise once (cta_sacc_collect).  Full range
// (R-24): a CTA that corrected products (X, one extended accumulator per dot)
// adds its normalised extended words into g[xs_off(ND) ..] and clears X.
template <int ND>
__device__ __forceinline__ void small_publish(CtaSacc<ND> &S, unsigned flags, long long *g, unsigned long long *X) {
    if (flags) atomicOr(&S.flags, flags);
    __syncthreads();
    for (int i = threadIdx.x; i < ND * SACC_L; i += blockDim.x) {
        const long long v = (long long)(&S.w[0][0])[i];
        if (v) atomicAdd((unsigned long long *)&g[i], (unsigned long long)v);
    }
    if (threadIdx.x == 0) {
        if (S.flags & FLAG_RANGE) atomicAdd((unsigned long long *)&g[ND * SACC_L], 1ull);
        if (S.flags & FLAG_NONFINITE) atomicAdd((unsigned long long *)&g[ND * SACC_L + 1], 1ull);
    }
    if ((S.flags & FLAG_RANGE) && X) {
        if (threadIdx.x < ND) xs_normalize((long long *)X + threadIdx.x * XS_L);
        __syncthreads();
        for (int i = threadIdx.x; i < ND * XS_L; i += blockDim.x) {
            if (X[i]) atomicAdd((unsigned long long *)&g[xs_off(ND) + i], X[i]);
            X[i] = 0ull;
        }
    }
}

// all CTAs: the words of one phase -> rounded dots -> the scalar step (every
// CTA reads the same buffer: its extended words are cleared by CTA 0 later)
template <int ND>
__device__ void small_round(CtaSacc<ND> &S, long long *g, int phase, Scalars *scl, double *hist) {
    if (threadIdx.x == 0) S.flags = 0u;
    unsigned gflags;
    cta_sacc_collect<ND>(S, g, gflags);
    const unsigned f = round_dots<ND>(S, g, gflags, phase_full_range(phase, scl), false);
    if (threadIdx.x == 0) phase_finalize(phase, scl, S.rounded, f, hist, nullptr, nullptr);
    __syncthreads();
}

// CTA 0 (all its threads): clear a phase buffer every CTA has read; its
// extended words only if some CTA wrote them (flag count != 0)
template <int ND>
__device__ __forceinline__ void small_clear(long long *g) {
    const bool ext = __ldcg(&g[ND * SACC_L]) != 0;
    __syncthreads();
    const int words = ext ? xs_words(ND) : ND * SACC_L + SACC_FLAGW;
    for (int i = threadIdx.x; i < words; i += blockDim.x) g[i] = 0;
}

// one product of the fused kernels: TwoProd + flag; a flagged product of
// finite operands is corrected into the dot's extended accumulator Xd when
// the solve runs with full range (R-24), a NaN/Inf operand flags NONFINITE
template <class TP>
__device__ __forceinline__ Prod small_prod(const TP &tp, double a, double b, bool zero_op, unsigned &flags,
                                           unsigned long long *Xd) {
    unsigned f = 0;
    const Prod P = tp.prep(a, b, zero_op, f);
    if (f) {
        if (!isfinite(a) || !isfinite(b)) f = FLAG_NONFINITE;
        else if (Xd) xs_correct(Xd, a, b);
        flags |= f;
    }
    return P;
}

// Plain dot mode (the paper's non-reproducible arm, NEXT-1): per-thread fma
// chains, a fixed xor-shuffle tree per warp, the warps summed in order into
// this CTA's partial part[blockIdx.x * ND + d] ...
template <int ND, int BS>
__device__ __forceinline__ void small_plain_publish(const double (&acc)[4], double *ws, double *part) {
#pragma unroll
    for (int d = 0; d < ND; ++d) {
        double v = acc[d];
#pragma unroll
        for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
        if ((threadIdx.x & 31) == 0) ws[(threadIdx.x >> 5) * 4 + d] = v;
    }
    __syncthreads();
    if (threadIdx.x < ND) {
        double t = 0.0;
        for (int w = 0; w < BS / 32; ++w) t = __dadd_rn(t, ws[w * 4 + threadIdx.x]);
        part[(size_t)blockIdx.x * ND + threadIdx.x] = t;
    }
}
// ... and, after the grid barrier, every CTA sums the partials in grid order
template <int ND>
__device__ void small_plain_round(const double *part, double *dsum, int phase, Scalars *scl, double *hist) {
    if (threadIdx.x < ND) {
        double t = 0.0;
        for (unsigned b = 0; b < gridDim.x; ++b) t = __dadd_rn(t, __ldcg(&part[(size_t)b * ND + threadIdx.x]));
        dsum[threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0) phase_finalize(phase, scl, dsum, 0u, hist, nullptr, nullptr);
    __syncthreads();
}

// this CTA's positions [P0, P1): y[row(pos)] = (A x)[row], the row's ordered fma chain (R-6)
__device__ __forceinline__ void small_spmv(const SmallArgs &a, int64_t P0, int64_t P1, const double *xb, double *yv) {
    for (int64_t pos = P0 + threadIdx.x; pos < P1; pos += blockDim.x) {
        const int64_t base = a.slice_off[pos >> 5] + (pos & 31);
        const int len = a.row_len[pos];
        double acc = 0.0;
        for (int k = 0; k < len; ++k)  // x written by other CTAs before the grid barrier: read through L2
            acc = __fma_rn(a.val[base + 32 * k], __ldcg(&xb[pos + a.col[base + 32 * k]]), acc);
        yv[a.perm ? (int64_t)a.perm[pos] : pos] = acc;
    }
}

// EXACT = false: plain fp64 dots (dot_mode PBCG_DOT_PLAIN); the partials go to
// gA[0] / gB[0] reinterpreted as doubles (G x 4 <= 256 of their 270 words)
template <int BS, bool EXACT>
__global__ void __launch_bounds__(BS, 1) pbcg_small_kernel(SmallArgs a) {
    __shared__ CtaSacc<4> SA;
    __shared__ CtaSacc<3> SB;
    __shared__ Scalars scs;
    __shared__ double ws[BS / 32 * 4], dsum[4];  // plain mode: warp sums, rounded dots
    __shared__ unsigned long long X[4 * XS_L];   // full range: extended accumulators of the corrected products
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t n = a.n;
    // whole sigma windows (256 rows) when rows are permuted, else whole slices
    const int64_t gran = a.perm ? 256 : 32, nw = (n + gran - 1) / gran;
    const int64_t P0 = min(n, gran * (nw * blockIdx.x / gridDim.x));
    const int64_t P1 = min(n, gran * (nw * (blockIdx.x + 1) / gridDim.x));
    Scalars *scl = blockIdx.x == 0 ? a.sc : &scs;  // CTA 0 keeps the global scalars and the history
    double *hist = blockIdx.x == 0 ? a.hist : nullptr;
    if (threadIdx.x == 0 && blockIdx.x != 0) scs = *a.sc;
    __syncthreads();
    const ExAccT<1, 1, 1> tp{};  // TwoProd + R-9 flag only
    // full range (R-24): corrections of flagged products go to X (per dot)
    const bool full = EXACT && scl->range_mode == 0;
    for (int i = threadIdx.x; i < 4 * XS_L; i += blockDim.x) X[i] = 0ull;
    __syncthreads();
    auto XD = [&](int d) -> unsigned long long * { return full ? X + d * XS_L : nullptr; };
    unsigned long long ts_prev = 0;
    (void)ts_prev;
    SMALL_TS(-1);
    for (int k = 0; k < a.iters && !scl->done; ++k) {
        const int par = scl->it & 1;
        // ---- K2 (l.70-74) + (q,y), (y,y), (r0,s), (r0,z) ----
        {
            const bool first = scl->it == 0;
            const double be = scl->beta, nom = -scl->omega, nal = -scl->alpha;
            unsigned flags = 0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};  // plain mode
            if (EXACT) cta_sacc_zero<4>(SA);
            __syncthreads();
            for (int64_t b0 = P0 + 32 * warp; b0 < P1; b0 += BS) {  // whole warps: the deposits are warp-wide
                const int64_t i = b0 + lane;
                const bool on = i < P1;
                Prod P[4] = {};
                if (on) {
                    const double r = a.r[i], w = a.w[i], t = a.t[i], rh = a.rh[i];
                    double p = r, s = w, z = t;  // beta_{-1} = 0: exact copies (R-3)
                    if (!first) {
                        const double v = a.v[i];
                        p = __fma_rn(be, __fma_rn(nom, a.s[i], a.p[i]), r);  // l.70
                        s = __fma_rn(be, __fma_rn(nom, a.z[i], a.s[i]), w);  // l.71
                        z = __fma_rn(be, __fma_rn(nom, v, a.z[i]), t);       // l.72
                    }
                    const double q = __fma_rn(nal, s, r), y = __fma_rn(nal, z, w);  // l.73-74
                    a.p[i] = p; a.s[i] = s; a.z[i] = z; a.q[i] = q; a.y[i] = y;
                    if (EXACT) {
                        const bool zy = is_zero(y), zr = is_zero(rh);
                        P[0] = small_prod(tp, q, y, is_zero(q) | zy, flags, XD(0));
                        P[1] = small_prod(tp, y, y, zy, flags, XD(1));
                        P[2] = small_prod(tp, rh, s, zr | is_zero(s), flags, XD(2));
                        P[3] = small_prod(tp, rh, z, zr | is_zero(z), flags, XD(3));
                    } else {
                        acc[0] = __fma_rn(q, y, acc[0]);
                        acc[1] = __fma_rn(y, y, acc[1]);
                        acc[2] = __fma_rn(rh, s, acc[2]);
                        acc[3] = __fma_rn(rh, z, acc[3]);
                    }
                }
                if (EXACT) {
#pragma unroll
                    for (int d = 0; d < 4; ++d) {  // one or two rows per lane: direct deposits (no warp aggregation chain)
                        if (is_nonzero(P[d].p)) sacc_deposit(SA.w[d], P[d].p);
                        if (is_nonzero(P[d].e)) sacc_deposit(SA.w[d], P[d].e);
                    }
                }
            }
            if (EXACT) small_publish<4>(SA, flags, a.gA[par], full ? X : nullptr);
            else small_plain_publish<4, BS>(acc, ws, (double *)a.gA[0]);
        }
        SMALL_TS(4);  // K2 rows + publish
        grid_barrier(a.bar);
        SMALL_TS(5);  // barrier A
        if (EXACT && blockIdx.x == 0) {  // every CTA has read gB of the previous iteration: clear it for the next one
            small_clear<3>(a.gB[par ^ 1]);
        }
        if (EXACT) small_round<4>(SA, a.gA[par], PH_A, scl, hist);  // l.76
        else small_plain_round<4>((const double *)a.gA[0], dsum, PH_A, scl, hist);
        SMALL_TS(6);  // round A
        if (scl->done) break;
        // ---- SpMV v = A z (l.75) over this CTA's rows ----
        small_spmv(a, P0, P1, a.zpad, a.v);
        __syncthreads();
        SMALL_TS(7);  // SpMV v
        // ---- K3 (l.77-79) + (r0,r'), (r0,w'), (r',r') ----
        {
            const double al = scl->alpha, om = scl->omega, nal = -al, nom = -om;
            unsigned flags = 0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};  // plain mode
            if (EXACT) cta_sacc_zero<3>(SB);
            __syncthreads();
            for (int64_t b0 = P0 + 32 * warp; b0 < P1; b0 += BS) {
                const int64_t i = b0 + lane;
                const bool on = i < P1;
                Prod P[3] = {};
                if (on) {
                    const double rh = a.rh[i], q = a.q[i], y = a.y[i];
                    const double x = __fma_rn(om, q, __fma_rn(al, a.p[i], a.x[i]));  // l.77
                    const double r = __fma_rn(nom, y, q);                            // l.78
                    const double w = __fma_rn(nom, __fma_rn(nal, a.v[i], a.t[i]), y);  // l.79
                    a.x[i] = x; a.r[i] = r; a.w[i] = w;
                    if (EXACT) {
                        const bool zr = is_zero(r), zh = is_zero(rh);
                        P[0] = small_prod(tp, rh, r, zh | zr, flags, XD(0));
                        P[1] = small_prod(tp, rh, w, zh | is_zero(w), flags, XD(1));
                        P[2] = small_prod(tp, r, r, zr, flags, XD(2));
                    } else {
                        acc[0] = __fma_rn(rh, r, acc[0]);
                        acc[1] = __fma_rn(rh, w, acc[1]);
                        acc[2] = __fma_rn(r, r, acc[2]);
                    }
                }
                if (EXACT) {
#pragma unroll
                    for (int d = 0; d < 3; ++d) {
                        if (is_nonzero(P[d].p)) sacc_deposit(SB.w[d], P[d].p);
                        if (is_nonzero(P[d].e)) sacc_deposit(SB.w[d], P[d].e);
                    }
                }
            }
            if (EXACT) small_publish<3>(SB, flags, a.gB[par], full ? X : nullptr);
            else small_plain_publish<3, BS>(acc, ws, (double *)a.gB[0]);
        }
        SMALL_TS(13);  // K3 rows + publish
        grid_barrier(a.bar);
        SMALL_TS(14);  // barrier B
        if (EXACT && blockIdx.x == 0) {  // every CTA has read gA of this iteration
            small_clear<4>(a.gA[par]);
        }
        if (EXACT) small_round<3>(SB, a.gB[par], PH_B, scl, hist);  // l.81-82, stopping and breakdown rules
        else small_plain_round<3>((const double *)a.gB[0], dsum, PH_B, scl, hist);
        if (scl->done) break;
        // ---- SpMV t = A w (l.80) ----
        small_spmv(a, P0, P1, a.wpad, a.t);
        __syncthreads();
        SMALL_TS(15);  // round B + SpMV t
    }
}

// Register-resident variant: rows not permuted, at most BS rows per CTA and at
// most 8 nonzeros per row (C1).  Thread t owns row P0 + t for the whole launch:
// its vector entries (x r r^ p s q y t v z w) and its SpMV row (values and
// x-buffer indices) stay in registers, so an iteration reads global memory
// only for the x gathers of the two SpMVs; z and w are stored as soon as they
// are formed (other CTAs gather them after the grid barrier), everything else
// once at exit.  Same arithmetic, same bits.
template <int BS, bool EXACT>
__global__ void __launch_bounds__(BS, 1) pbcg_small_reg_kernel(SmallArgs a) {
    __shared__ CtaSacc<4> SA;
    __shared__ CtaSacc<3> SB;
    __shared__ Scalars scs;
    __shared__ double ws[BS / 32 * 4], dsum[4];
    __shared__ unsigned long long X[4 * XS_L];
    // a launch enqueued after the solve stopped (the overlapped polls of
    // pbicgstab_solve): no reload and store-back of the state
    if (__ldcg(&a.sc->done)) return;
    const int64_t n = a.n, nw = (n + 31) / 32;
    const int64_t P0 = min(n, 32 * (nw * blockIdx.x / gridDim.x));
    const int64_t P1 = min(n, 32 * (nw * (blockIdx.x + 1) / gridDim.x));
    Scalars *scl = blockIdx.x == 0 ? a.sc : &scs;
    double *hist = blockIdx.x == 0 ? a.hist : nullptr;
    if (threadIdx.x == 0 && blockIdx.x != 0) scs = *a.sc;
    const int64_t i = P0 + threadIdx.x;
    const bool on = i < P1;
    double x = 0, r = 0, rh = 0, p = 0, s = 0, q = 0, y = 0, t = 0, v = 0, z = 0, w = 0;
    double mv[8];
    int64_t mx[8];
    int len = 0;
    if (on) {
        x = a.x[i]; r = a.r[i]; rh = a.rh[i]; p = a.p[i]; s = a.s[i]; q = a.q[i]; y = a.y[i];
        t = a.t[i]; v = a.v[i]; z = a.z[i]; w = a.w[i];
        const int64_t base = a.slice_off[i >> 5] + (i & 31);
        len = a.row_len[i];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            mv[k] = k < len ? a.val[base + 32 * k] : 0.0;
            mx[k] = k < len ? i + a.col[base + 32 * k] : 0;
        }
    }
    __syncthreads();
    const ExAccT<1, 1, 1> tp{};
    // full range (R-24): corrections of flagged products go to X (per dot)
    const bool full = EXACT && scl->range_mode == 0;
    for (int i = threadIdx.x; i < 4 * XS_L; i += blockDim.x) X[i] = 0ull;
    __syncthreads();
    auto XD = [&](int d) -> unsigned long long * { return full ? X + d * XS_L : nullptr; };
    bool k3_done = true;  // the registers hold the state after K3 (or at entry)
    for (int k = 0; k < a.iters && !scl->done; ++k) {
        const int par = scl->it & 1;
        // ---- K2 (l.70-74) ----
        {
            const bool first = scl->it == 0;
            const double be = scl->beta, nom = -scl->omega, nal = -scl->alpha;
            unsigned flags = 0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (EXACT) cta_sacc_zero<4>(SA);
            __syncthreads();
            Prod P[4] = {};
            if (on) {
                if (first) {  // beta_{-1} = 0: exact copies (R-3)
                    p = r; s = w; z = t;
                } else {
                    const double sp = s, zp = z;
                    p = __fma_rn(be, __fma_rn(nom, sp, p), r);  // l.70
                    s = __fma_rn(be, __fma_rn(nom, zp, sp), w);  // l.71
                    z = __fma_rn(be, __fma_rn(nom, v, zp), t);   // l.72
                }
                q = __fma_rn(nal, s, r);  // l.73
                y = __fma_rn(nal, z, w);  // l.74
                a.z[i] = z;               // gathered by the SpMV of every CTA
                if (EXACT) {
                    const bool zy = is_zero(y), zr = is_zero(rh);
                    P[0] = small_prod(tp, q, y, is_zero(q) | zy, flags, XD(0));
                    P[1] = small_prod(tp, y, y, zy, flags, XD(1));
                    P[2] = small_prod(tp, rh, s, zr | is_zero(s), flags, XD(2));
                    P[3] = small_prod(tp, rh, z, zr | is_zero(z), flags, XD(3));
                } else {
                    acc[0] = __fma_rn(q, y, 0.0);
                    acc[1] = __fma_rn(y, y, 0.0);
                    acc[2] = __fma_rn(rh, s, 0.0);
                    acc[3] = __fma_rn(rh, z, 0.0);
                }
            }
            k3_done = false;
            if (EXACT) {
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    if (is_nonzero(P[d].p)) sacc_deposit(SA.w[d], P[d].p);
                    if (is_nonzero(P[d].e)) sacc_deposit(SA.w[d], P[d].e);
                }
                small_publish<4>(SA, flags, a.gA[par], full ? X : nullptr);
            } else {
                small_plain_publish<4, BS>(acc, ws, (double *)a.gA[0]);
            }
        }
        grid_barrier(a.bar);
        if (EXACT && blockIdx.x == 0)
            small_clear<3>(a.gB[par ^ 1]);
        if (EXACT) small_round<4>(SA, a.gA[par], PH_A, scl, hist);  // l.76
        else small_plain_round<4>((const double *)a.gA[0], dsum, PH_A, scl, hist);
        if (scl->done) break;
        // ---- SpMV v = A z (l.75): the row's ordered fma chain (R-6) ----
        if (on) {
            double sum = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                if (kk < len) sum = __fma_rn(mv[kk], __ldcg(&a.zpad[mx[kk]]), sum);  // other CTAs' z: L2
            v = sum;
        }
        // ---- K3 (l.77-79) ----
        {
            const double al = scl->alpha, om = scl->omega, nal = -al, nom = -om;
            unsigned flags = 0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (EXACT) cta_sacc_zero<3>(SB);
            __syncthreads();
            Prod P[3] = {};
            if (on) {
                x = __fma_rn(om, q, __fma_rn(al, p, x));       // l.77
                r = __fma_rn(nom, y, q);                        // l.78
                w = __fma_rn(nom, __fma_rn(nal, v, t), y);      // l.79
                a.w[i] = w;
                if (EXACT) {
                    const bool zr = is_zero(r), zh = is_zero(rh);
                    P[0] = small_prod(tp, rh, r, zh | zr, flags, XD(0));
                    P[1] = small_prod(tp, rh, w, zh | is_zero(w), flags, XD(1));
                    P[2] = small_prod(tp, r, r, zr, flags, XD(2));
                } else {
                    acc[0] = __fma_rn(rh, r, 0.0);
                    acc[1] = __fma_rn(rh, w, 0.0);
                    acc[2] = __fma_rn(r, r, 0.0);
                }
            }
            k3_done = true;
            if (EXACT) {
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    if (is_nonzero(P[d].p)) sacc_deposit(SB.w[d], P[d].p);
                    if (is_nonzero(P[d].e)) sacc_deposit(SB.w[d], P[d].e);
                }
                small_publish<3>(SB, flags, a.gB[par], full ? X : nullptr);
            } else {
                small_plain_publish<3, BS>(acc, ws, (double *)a.gB[0]);
            }
        }
        grid_barrier(a.bar);
        if (EXACT && blockIdx.x == 0)
            small_clear<4>(a.gA[par]);
        if (EXACT) small_round<3>(SB, a.gB[par], PH_B, scl, hist);
        else small_plain_round<3>((const double *)a.gB[0], dsum, PH_B, scl, hist);
        if (scl->done) break;
        // ---- SpMV t = A w (l.80) ----
        if (on) {
            double sum = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                if (kk < len) sum = __fma_rn(mv[kk], __ldcg(&a.wpad[mx[kk]]), sum);
            t = sum;
        }
    }
    (void)k3_done;
    if (on) {  // the state back to global memory (z and w are there already)
        a.x[i] = x; a.r[i] = r; a.p[i] = p; a.s[i] = s; a.q[i] = q; a.y[i] = y; a.t[i] = t; a.v[i] = v;
    }
}

}  // namespace pbcg
