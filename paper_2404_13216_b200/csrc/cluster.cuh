// cluster.cuh -- the whole p-BiCGStab iteration (Alg. 2 l.70-82) for small
// systems in ONE thread-block cluster (C1: 4,096 rows = 16 CTAs x 256 rows).
//
// B200 design (DESIGN.md §5 "Cluster kernel"): the fused small kernel
// (small.cuh) synchronises its grid through global-memory atomics (~2 us per
// barrier) and exchanges z, w and the dot partials through L2.  Here the
// grid IS one cluster of CL CTAs (CL = 16, non-portable size; 8 if the
// device cannot schedule 16):
//   * thread t of CTA c owns row c R + t for the whole launch (R rows per
//     CTA, whole 32-row slices); its vector entries and its SpMV row stay in
//     registers, as in pbcg_small_reg_kernel;
//   * z and w of the own rows live in the CTA's shared memory; the SpMV
//     gathers them from the owning CTA through distributed shared memory
//     (DSMEM, generic pointers from map_shared_rank);
//   * every CTA deposits its products into its own superaccumulator (shared
//     atomics), then red.adds its nonzero words into CTA 0's phase buffer
//     over DSMEM; barrier.cluster (release/acquire) replaces the grid
//     barrier; every CTA copies the summed words from CTA 0, normalises,
//     rounds (RN-even; the R-24 extended words when flagged) and runs the
//     scalar step on its own copy (CTA 0: the global scalars + history).
// The arithmetic is that of the six-kernel path element by element (FMA
// policy F, the per-row fma chain, exact dots): the same bits.
#pragma once
#include <cooperative_groups.h>

#include "small.cuh"

namespace pbcg {

namespace cgx = cooperative_groups;

// phase buffer words (4 dots: PH_A, 3 dots: PH_B) incl. the extended words of R-24
constexpr int CLA_WORDS = xs_words(4), CLB_WORDS = xs_words(3);

// The dots of a phase from a local copy `g` of CTA 0's summed fast words and
// flag counts (not normalised): normalise, round (warp per dot), and when some
// CTA flagged a product (full range, R-24) the extended words, read from CTA
// 0's buffer `gext` itself (DSMEM).  Returns the flags for
// phase_finalize (as round_dots).  All threads.
template <int ND>
__device__ unsigned cluster_round(CtaSacc<ND> &S, const long long *g, const long long *gext, bool full) {
    long long *w = (long long *)&S.w[0][0];
    for (int i = threadIdx.x; i < ND * SACC_L; i += blockDim.x) w[i] = g[i];
    __syncthreads();
    if (threadIdx.x < ND) sacc_normalize(w + threadIdx.x * SACC_L);
    __shared__ unsigned ovf;
    if (threadIdx.x == 0) ovf = 0u;
    __syncthreads();
    const unsigned gflags = (g[ND * SACC_L] ? FLAG_RANGE : 0u) | (g[ND * SACC_L + 1] ? FLAG_NONFINITE : 0u);
    if ((threadIdx.x >> 5) < ND) {
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
    if (gflags & FLAG_NONFINITE) return FLAG_NONFINITE;
    __shared__ long long X[XS_L];
    unsigned o2 = 0u;
    for (int d = 0; d < ND; ++d) {
        for (int i = threadIdx.x; i < XS_L; i += blockDim.x) X[i] = gext[xs_off(ND) + d * XS_L + i];
        __syncthreads();
        if (threadIdx.x == 0) {
            const long long *wd = w + d * SACC_L;
            for (int i = 0; i < SACC_L; ++i) X[i + 33] += wd[i] * (1ll << 18);  // 2^-1074 = extended bit 1074
            xs_normalize(X);
            const double v = xs_round(X);
            S.rounded[d] = v;
            if (isinf(v)) o2 |= FLAG_RANGE;
        }
        __syncthreads();
    }
    return o2;
}

// The lanes deposit their products into CL_NCOPY copies of the CTA's
// superaccumulator (lane % CL_NCOPY): lanes of similar exponents hit the same
// few words, and the shared atomics of one word serialise.
constexpr int CL_NCOPY = 8;

// This CTA's words (the sum of the lane copies cp[copy][d][word], which are
// cleared for the next phase), flag counts and extended words into CTA 0's
// phase buffer g0 (a DSMEM pointer): nonzero words only.  All threads.
template <int ND>
__device__ __forceinline__ void cluster_publish(unsigned &cflags, unsigned flags, unsigned long long *cp, long long *g0,
                                                unsigned long long *X) {
    if (flags) atomicOr(&cflags, flags);
    __syncthreads();
    for (int j = threadIdx.x; j < ND * SACC_L; j += blockDim.x) {
        const int d = j / SACC_L, wi = j - d * SACC_L;
        long long v = 0;
#pragma unroll
        for (int c = 0; c < CL_NCOPY; ++c) {
            unsigned long long &cw = cp[(c * 4 + d) * SACC_L + wi];
            v += (long long)cw;
            cw = 0ull;
        }
        if (v) atomicAdd((unsigned long long *)&g0[j], (unsigned long long)v);
    }
    if (threadIdx.x == 0) {
        if (cflags & FLAG_RANGE) atomicAdd((unsigned long long *)&g0[ND * SACC_L], 1ull);
        if (cflags & FLAG_NONFINITE) atomicAdd((unsigned long long *)&g0[ND * SACC_L + 1], 1ull);
    }
    if ((cflags & FLAG_RANGE) && X) {  // full range: the corrected products' extended words
        if (threadIdx.x < ND) xs_normalize((long long *)X + threadIdx.x * XS_L);
        __syncthreads();
        for (int i = threadIdx.x; i < ND * XS_L; i += blockDim.x) {
            if (X[i]) atomicAdd((unsigned long long *)&g0[xs_off(ND) + i], X[i]);
            X[i] = 0ull;
        }
    }
}

// Plain dot mode: this CTA's partials (warp sums in order) into CTA 0's part[c][d]
template <int ND, int BS>
__device__ __forceinline__ void cluster_plain_publish(const double (&acc)[4], double *ws, double *part0) {
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
        part0[(size_t)blockIdx.x * 4 + threadIdx.x] = t;
    }
}

// dynamic shared memory of the cluster kernel (8-byte words)
template <int BS>
struct ClusterSmem {
    static constexpr int GA = 0;                            // long long gA[2][CLA_WORDS] (CTA 0's: the cluster's)
    static constexpr int GB = GA + 2 * CLA_WORDS;           // long long gB[2][CLB_WORDS]
    static constexpr int GL = GB + 2 * CLB_WORDS;           // long long gl[ND SACC_L + FLAGW]: local copy
    static constexpr int XX = GL + 4 * SACC_L + SACC_FLAGW;  // ull X[4][XS_L]: corrections (R-24)
    static constexpr int CP = XX + 4 * XS_L;                // ull cp[CL_NCOPY][4][SACC_L]: lane copies
    static constexpr int ZS = CP + CL_NCOPY * 4 * SACC_L;   // double zs[BS], wsv[BS]: z, w of the own rows
    static constexpr int PT = ZS + 2 * BS;                  // double part[2][16][4]: plain mode partials (CTA 0's)
    static constexpr int WORDS = PT + 2 * 16 * 4;
    static constexpr size_t BYTES = 8 * (size_t)WORDS;
};

// BS threads per CTA (one row each), CL CTAs = one cluster (the whole grid)
template <int BS, bool EXACT>
__global__ void __launch_bounds__(BS, 1) pbcg_cluster_kernel(SmallArgs a) {
    using L = ClusterSmem<BS>;
    __shared__ CtaSacc<4> SA;
    __shared__ CtaSacc<3> SB;
    __shared__ Scalars scs;
    __shared__ double wsum[BS / 32 * 4], dsum[4];
    extern __shared__ __align__(16) unsigned long long dsm[];
    long long(*gA)[CLA_WORDS] = (long long(*)[CLA_WORDS])(dsm + L::GA);
    long long(*gB)[CLB_WORDS] = (long long(*)[CLB_WORDS])(dsm + L::GB);
    long long *gl = (long long *)(dsm + L::GL);
    unsigned long long *X = dsm + L::XX, *cp = dsm + L::CP;
    double *zs = (double *)(dsm + L::ZS), *wsv = zs + BS, *part = (double *)(dsm + L::PT);
    cgx::cluster_group cl = cgx::this_cluster();
    if (__ldcg(&a.sc->done)) return;  // every CTA: the same value (the solve stopped before this launch)
    const int c = (int)cl.block_rank(), CL = (int)cl.num_blocks();
    const int64_t n = a.n, nw = (n + 31) / 32;
    const int64_t R = 32 * ((nw + CL - 1) / CL);  // rows per CTA (whole slices); owner(g) = g / R
    const int64_t P0 = min(n, R * c), P1 = min(n, R * (c + 1));
    const int64_t own_off = a.z - a.zpad;          // x-buffer index of row 0
    Scalars *scl = c == 0 ? a.sc : &scs;
    double *hist = c == 0 ? a.hist : nullptr;
    if (threadIdx.x == 0 && c != 0) scs = *a.sc;
    for (int j = threadIdx.x; j < L::ZS; j += BS) dsm[j] = 0ull;  // phase buffers, copies, corrections
    const int64_t i = P0 + threadIdx.x;
    const bool on = i < P1;
    double x = 0, r = 0, rh = 0, p = 0, s = 0, q = 0, y = 0, t = 0, v = 0, z = 0, w = 0;
    double mv[8];
    const double *mz[8];  // the gathered z entries: (CTA, offset) of each column, as DSMEM pointers
    int len = 0;
    if (on) {
        x = a.x[i]; r = a.r[i]; rh = a.rh[i]; p = a.p[i]; s = a.s[i]; q = a.q[i]; y = a.y[i];
        t = a.t[i]; v = a.v[i]; z = a.z[i]; w = a.w[i];
    }
    zs[threadIdx.x] = z;
    wsv[threadIdx.x] = w;
    if (on) {
        const int64_t base = a.slice_off[i >> 5] + (i & 31);
        len = a.row_len[i];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            mv[k] = k < len ? a.val[base + 32 * k] : 0.0;
            const int64_t g = k < len ? i + a.col[base + 32 * k] - own_off : i;  // the column's row
            mz[k] = cl.map_shared_rank(zs, (unsigned)(g / R)) + (g % R);
        }
    }
    const ExAccT<1, 1, 1> tp{};
    const bool full = EXACT && scl->range_mode == 0;
    auto XD = [&](int d) -> unsigned long long * { return full ? X + d * XS_L : nullptr; };
    long long *gA0[2] = {cl.map_shared_rank(&gA[0][0], 0u), cl.map_shared_rank(&gA[1][0], 0u)};
    long long *gB0[2] = {cl.map_shared_rank(&gB[0][0], 0u), cl.map_shared_rank(&gB[1][0], 0u)};
    double *part0 = cl.map_shared_rank(part, 0u);
    cl.sync();  // every CTA's zs, ws and zeroed buffers in place
    const ptrdiff_t w_off = wsv - zs;  // the w gathers: same CTA and offset, the other array
    unsigned long long ts_prev = 0;
    (void)ts_prev;
    SMALL_TS(-1);
    for (int k = 0; k < a.iters && !scl->done; ++k) {
        const int par = scl->it & 1;
        // ---- K2 (l.70-74) ----
        {
            const bool first = scl->it == 0;
            const double be = scl->beta, nom = -scl->omega, nal = -scl->alpha;
            unsigned flags = 0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (threadIdx.x == 0) SA.flags = 0u;
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
                zs[threadIdx.x] = z;      // gathered by the SpMV of every CTA (DSMEM)
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
            if (EXACT) {
                unsigned long long *mine = cp + (threadIdx.x & (CL_NCOPY - 1)) * 4 * SACC_L;
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                    if (is_nonzero(P[d].p)) sacc_deposit(mine + d * SACC_L, P[d].p);
                    if (is_nonzero(P[d].e)) sacc_deposit(mine + d * SACC_L, P[d].e);
                }
                cluster_publish<4>(SA.flags, flags, cp, gA0[par], full ? X : nullptr);
            } else {
                cluster_plain_publish<4, BS>(acc, wsum, part0);
            }
        }
        SMALL_TS(4);
        cl.sync();  // z of every row and every CTA's words are complete (release / acquire)
        SMALL_TS(5);
        // ---- round phase A (l.76): every CTA from a local copy of CTA 0's words ----
        if (EXACT) {
            const long long *src = gA0[par];
            for (int j = threadIdx.x; j < 4 * SACC_L + SACC_FLAGW; j += BS) gl[j] = src[j];
            __syncthreads();
            const unsigned f = cluster_round<4>(SA, gl, src, phase_full_range(PH_A, scl));
            if (threadIdx.x == 0) phase_finalize(PH_A, scl, SA.rounded, f, hist, nullptr, nullptr);
        } else {
            if (threadIdx.x < 4) {
                double tt = 0.0;
                for (int b = 0; b < CL; ++b) tt = __dadd_rn(tt, part0[b * 4 + threadIdx.x]);
                dsum[threadIdx.x] = tt;
            }
            __syncthreads();
            if (threadIdx.x == 0) phase_finalize(PH_A, scl, dsum, 0u, hist, nullptr, nullptr);
        }
        __syncthreads();
        if (EXACT && c == 0)  // every CTA read gB of the previous iteration before this barrier
            for (int j = threadIdx.x; j < CLB_WORDS; j += BS) gB[par ^ 1][j] = 0;
        SMALL_TS(6);
        if (scl->done) break;
        // ---- SpMV v = A z (l.75): the row's ordered fma chain (R-6), z over DSMEM ----
        if (on) {
            double sum = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                if (kk < len) sum = __fma_rn(mv[kk], *mz[kk], sum);
            v = sum;
        }
        SMALL_TS(7);
        // ---- K3 (l.77-79) ----
        {
            const double al = scl->alpha, om = scl->omega, nal = -al, nom = -om;
            unsigned flags = 0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
            if (threadIdx.x == 0) SB.flags = 0u;
            __syncthreads();
            Prod P[3] = {};
            if (on) {
                x = __fma_rn(om, q, __fma_rn(al, p, x));   // l.77
                r = __fma_rn(nom, y, q);                    // l.78
                w = __fma_rn(nom, __fma_rn(nal, v, t), y);  // l.79
                wsv[threadIdx.x] = w;
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
            if (EXACT) {
                unsigned long long *mine = cp + (threadIdx.x & (CL_NCOPY - 1)) * 4 * SACC_L;
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    if (is_nonzero(P[d].p)) sacc_deposit(mine + d * SACC_L, P[d].p);
                    if (is_nonzero(P[d].e)) sacc_deposit(mine + d * SACC_L, P[d].e);
                }
                cluster_publish<3>(SB.flags, flags, cp, gB0[par], full ? X : nullptr);
            } else {
                cluster_plain_publish<3, BS>(acc, wsum, part0 + 64);  // phase B partials: the second half
            }
        }
        SMALL_TS(13);
        cl.sync();
        SMALL_TS(14);
        // ---- round phase B (l.81-82, stopping and breakdown rules) ----
        if (EXACT) {
            const long long *src = gB0[par];
            for (int j = threadIdx.x; j < 3 * SACC_L + SACC_FLAGW; j += BS) gl[j] = src[j];
            __syncthreads();
            const unsigned f = cluster_round<3>(SB, gl, src, phase_full_range(PH_B, scl));
            if (threadIdx.x == 0) phase_finalize(PH_B, scl, SB.rounded, f, hist, nullptr, nullptr);
        } else {
            if (threadIdx.x < 3) {
                double tt = 0.0;
                for (int b = 0; b < CL; ++b) tt = __dadd_rn(tt, part0[64 + b * 4 + threadIdx.x]);
                dsum[threadIdx.x] = tt;
            }
            __syncthreads();
            if (threadIdx.x == 0) phase_finalize(PH_B, scl, dsum, 0u, hist, nullptr, nullptr);
        }
        __syncthreads();
        if (EXACT && c == 0)  // every CTA read gA of this iteration before this barrier
            for (int j = threadIdx.x; j < CLA_WORDS; j += BS) gA[par][j] = 0;
        if (scl->done) break;
        // ---- SpMV t = A w (l.80) ----
        if (on) {
            double sum = 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk)
                if (kk < len) sum = __fma_rn(mv[kk], *(mz[kk] + w_off), sum);
            t = sum;
        }
        SMALL_TS(15);
    }
    if (on) {  // the state back to global memory
        a.x[i] = x; a.r[i] = r; a.p[i] = p; a.s[i] = s; a.q[i] = q; a.y[i] = y; a.t[i] = t; a.v[i] = v;
        a.z[i] = z; a.w[i] = w;
    }
    cl.sync();  // no CTA leaves while others may still read its shared memory
}

}  // namespace pbcg
