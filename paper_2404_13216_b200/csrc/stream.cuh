// stream.cuh -- persistent, warp-specialised streaming kernels for the
// vector part of p-BiCGStab (K2, K3) and for the standalone EXDOT.
//
// B200 design: one CTA per SM; one producer warp streams tiles
// of every input vector HBM -> shared memory with cp.async.bulk (the TMA bulk
// engine, SASS UBLKCP) into a STAGES-deep ring guarded by mbarriers
// (full: transaction bytes landed; empty: every consumer warp is done);
// NCW consumer warps read their rows from shared memory, run the recurrences
// and the ExBLAS accumulation in registers, and store the output vectors with
// coalesced 16-byte stores.  Memory stays busy while the fp64 pipe works on
// the previous tiles, so the kernel runs at max(HBM time, fp64 time) instead
// of their sum, without spending registers on loads in flight.
#pragma once
#include <cstdint>
#include <type_traits>

#include "kernels.cuh"

// One cold-tier vote per (dot, stream) instead of per stream in the two-dot
// groups (cascade_batch SPLIT), by kernel and cold depth NL.  On in K3,
// whose group 0 pairs a dot that spills often, (r0,r'), with one that rarely
// does, (r',r'): C5 1,071.5 -> 1,080.4 iter/s at the driver's K = 20
// (1,084.5 -> 1,091.6 at K = 200); off in K2 (both pairs spill alike: C5
// 1,068.7, C3 7,724 vs 7,770; lean K2 with it C3 8,491 vs 8,536;
// tools/ab_iter.py).
#ifndef PBCG_VSPLIT_K2
#define PBCG_VSPLIT_K2(nl) false
#endif
#ifndef PBCG_VSPLIT_K3
#define PBCG_VSPLIT_K3(nl) true  // the lean / pipelined K3 (one cold level) too: C3 8,512 -> 8,536, C4 and the bjacobi2_pipe arm unchanged
#endif

namespace pbcg {

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// 1-D bulk copy global -> shared (TMA bulk engine), completion counted on bar
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

// The same with the L2 evict_first priority: the matrix streams of the SpMV
// kernels.  A matrix chunk is read once per SpMV and is larger than what the
// L2 could keep until the next one, so without the hint it only pushes out
// the vectors the neighbouring kernels re-read (K2's z is the next SpMV's x,
// v and t are K3's and K2's inputs).  tools/ab_iter.py: C3 (16.8 MB vectors,
// 134 MB matrix, 126 MB L2) 7,766 -> 8,207 iter/s, C5 1,082 -> 1,090.
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s_stream(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

__device__ __forceinline__ void st_stream_v2(double2 *p, double2 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x), "d"(v.y), "l"(pol) : "memory");
}
// Vectors that K2 / K3 stream through the L2 with the evict_first hint, loads
// (EFM: bit v = ring vector v) and stores (STM: K2 p,s,z,q,y / K3 x,r,w).
// Default: s (touched by K2 only) and x (K3 only) -- their next use is a whole
// iteration away, so they only take the cache from vectors the next kernel
// reads.  tools/ab_iter.py on top of the matrix hint: C5 1,090.7 -> 1,096.9
// iter/s, C3 8,213 -> 8,223, C4 unchanged.  Measured and rejected: every
// load and store (C5 1,076.5, C3 8,061), everything but the SpMV inputs z, w
// (1,077.9 / 8,150), s, p, r0 / x, p, r0 (1,093.5 / 8,203), stores only
// (1,089.7 / 8,117), and the loads of the vectors the next kernel overwrites
// (r, w, v / q, y, t: C3 8,163 vs 8,206 -- their dirty lines then go to DRAM
// instead of being overwritten in the cache).
#ifndef PBCG_K2_EFM
#define PBCG_K2_EFM 0x20u
#endif
#ifndef PBCG_K3_EFM
#define PBCG_K3_EFM 0x40u
#endif
// Vectors whose K2 / K3 loads carry evict_last (ELM, same bit order as EFM): K2's r0 (the shadow residual, read
// by K2 and K3 in every iteration and never written), p and z (read here, overwritten in place, re-read by K3 / the
// SpMV).  tools/ab_iter.py: C3 8,405 -> 8,513 iter/s, C5 1,097.8 -> 1,100.3; r0 alone 8,460, r0 + p 8,504 (C4 1,604
// -> 1,614), r0 + t 8,457, r0 + t + v 8,460; with K3's p / r0 / both as well 8,504 / 8,480 / 8,435.  evict_last on
// STORES loses everywhere (z; z, q, y; K3's w; z and w; p, z: C3 8,457-8,497 vs 8,514, C5 1,080-1,094 vs 1,101).
#ifndef PBCG_K2_ELM
#define PBCG_K2_ELM 0x52u
#endif
#ifndef PBCG_K3_ELM
#define PBCG_K3_ELM 0u
#endif
#ifndef PBCG_K2_STM
#define PBCG_K2_STM 0x2u
#endif
#ifndef PBCG_K3_STM
#define PBCG_K3_STM 0x1u
#endif
template <unsigned M, int B>
__device__ __forceinline__ void st_v2(double *base, int64_t gp, double2 v, uint64_t pol) {
    if constexpr ((M >> B) & 1u) st_stream_v2((double2 *)base + gp, v, pol);
    else ((double2 *)base)[gp] = v;
}

// Tile geometry shared by the producer and the consumers.
template <int NCW, int PPT>
struct TileGeo {
    static constexpr int PAIRS = NCW * 32 * PPT;  // row pairs per tile
    static constexpr int T = 2 * PAIRS;           // rows per tile
};

// Producer loop (one lane): for each tile owned by this CTA, wait for a free
// slot, arm the full barrier with the byte count and issue one bulk copy per
// input vector.  Rows are copied in whole pairs (16-byte multiples); an odd
// last row is read directly from global memory by its consumer.
template <int NV, int T, int STAGES>
__device__ __forceinline__ void produce(const double *const *src, int nv_act, int64_t n, double *buf, uint64_t *full,
                                        uint64_t *empty) {
    const int64_t ntiles = (n + T - 1) / T;
    int s = 0;
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        mbar_wait(&empty[s], ph ^ 1u);
        const int64_t r0 = tile * T;
        const int rows = (int)min((int64_t)T, n - r0);
        const uint32_t bytes = (uint32_t)(rows & ~1) * 8u;
        mbar_expect_tx(&full[s], bytes * (uint32_t)nv_act);
        if (bytes) {
#pragma unroll
            for (int v = 0; v < NV; ++v)  // static indices keep src in registers
                if (v < nv_act) bulk_g2s(buf + ((size_t)s * NV + v) * T, src[v] + r0, bytes, &full[s]);
        }
        if (++s == STAGES) { s = 0; ph ^= 1u; }
    }
}

// Ring stages issued before the PDL gate (K2 / K3).  Issuing all of them
// makes the first tile wait for the whole burst (no priority among bulk
// copies); fewer stages let the first tiles land sooner after the gate.
#ifndef PBCG_PREGATE
#define PBCG_PREGATE 2  // C3: 7,404 (all 5) -> 7,582 iter/s (1), C5 1,111 -> 1,116; with the L2 hints 2 stages: C3 8,377 -> 8,410, C5 / C4 +0.1 % (tools/ab_iter.py)
#endif
#define PBCG_PREGATE_STAGES(S) ((PBCG_PREGATE) < (S) ? (PBCG_PREGATE) : (S))

// The same, for a kernel launched with PDL: the first STAGES tiles of every
// vector except `late` (the one the immediately preceding kernel writes) are
// issued before `gate` (which waits on that kernel and returns false to
// abort); every earlier kernel of the stream has completed by the time this
// one launches.  The late vector's copies of those tiles follow the gate
// (their bytes are already in the barrier's expected count); on abort they
// are issued anyway and drained, so no copy is in flight at exit.
// EFM: bit v set = vector v streams through the L2 (evict_first hint).
template <int NV, int T, int STAGES, unsigned EFM = 0u, unsigned ELM = 0u, class Gate>
__device__ __forceinline__ bool produce_gated(const double *const *src, int nv_act, int late, int64_t n, double *buf,
                                              uint64_t *full, uint64_t *empty, Gate gate) {
    [[maybe_unused]] const uint64_t pol = EFM ? l2_policy_evict_first() : 0ull;
    [[maybe_unused]] uint64_t pol_last = 0ull;
    if constexpr (ELM != 0u) asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol_last));
    const int64_t ntiles = (n + T - 1) / T;
    int s = 0, issued = 0;
    uint32_t ph = 0;
    bool gated = false;
    auto tile_bytes = [&](int64_t tile) { return (uint32_t)((int)min((int64_t)T, n - tile * T) & ~1) * 8u; };
    auto open_gate = [&]() {
        gated = true;
        const bool ok = gate();
        if (late >= 0 && late < nv_act) {
            const double *sl = nullptr;
#pragma unroll
            for (int v = 0; v < NV; ++v)  // static indices keep src in registers
                if (v == late) sl = src[v];
            for (int k = 0; k < issued; ++k) {  // first pass: ring stage k holds tile blockIdx.x + k gridDim.x
                const int64_t tile = blockIdx.x + (int64_t)k * gridDim.x;
                const uint32_t by = tile_bytes(tile);
                if (by) bulk_g2s(buf + ((size_t)k * NV + late) * T, sl + tile * T, by, &full[k]);
            }
        }
        if (!ok)
            for (int k = 0; k < issued; ++k) mbar_wait(&full[k], 0u);
        return ok;
    };
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        if (!gated && issued == PBCG_PREGATE_STAGES(STAGES) && !open_gate()) return false;
        mbar_wait(&empty[s], ph ^ 1u);
        const int64_t r0 = tile * T;
        const uint32_t bytes = tile_bytes(tile);
        mbar_expect_tx(&full[s], bytes * (uint32_t)nv_act);
        if (bytes) {
#pragma unroll
            for (int v = 0; v < NV; ++v)  // static indices keep src in registers
                if (v < nv_act && (gated || v != late)) {
                    if ((EFM >> v) & 1u) bulk_g2s_stream(buf + ((size_t)s * NV + v) * T, src[v] + r0, bytes, &full[s], pol);
                    else if ((ELM >> v) & 1u) bulk_g2s_stream(buf + ((size_t)s * NV + v) * T, src[v] + r0, bytes, &full[s], pol_last);
                    else bulk_g2s(buf + ((size_t)s * NV + v) * T, src[v] + r0, bytes, &full[s]);
                }
        }
        ++issued;
        if (++s == STAGES) { s = 0; ph ^= 1u; }
    }
    return gated ? true : open_gate();
}

template <int NV, int T, int STAGES>
__device__ __forceinline__ size_t stream_smem_bytes() {
    return sizeof(double) * (size_t)STAGES * NV * T + 2 * STAGES * sizeof(uint64_t);
}

// End of a dot-split stream kernel (exact dots): every consumer warp drains
// its two accumulators into its own words of the drained ring (plain adds,
// warp_deposit_priv), then the CTA adds the warps' words into S.w -- the
// shared-atomic storm of all warps depositing into the same few words of S.w
// (measured: 6-8 us per launch on C3) is gone.  dot(g, k): the dot of
// accumulator k of dot group g, or -1.  All threads.
// The drain goes through a per-warp window (warp_window_deposit) instead of
// one warp-aggregated deposit per term: tools/ab_iter.py, C3 8,222 -> 8,338
// iter/s, C4 1,612 -> 1,617, C5 1,097 -> 1,098 (windows of 10 / 16 / 24 words
// alike).  Ring memory used: drain_ring_words int64.
#ifndef PBCG_WIN_DRAIN
#define PBCG_WIN_DRAIN 1
#endif
__host__ __device__ constexpr size_t drain_ring_words(int nwarps) { return (size_t)nwarps * (2 * SACC_L + (PBCG_WIN_DRAIN ? WIN_WORDS : 0)); }
template <int ND, int NCW, int W, class Acc, class Dot>
__device__ __forceinline__ void drain_private(CtaSacc<ND> &S, Acc &d0, Acc &d1, long long *ring, Dot dot) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __syncthreads();  // every consumer is done with the ring
    PBCG_TL(ND == 4 ? 0 : 2, 6);
    long long *pw = ring + (size_t)warp * 2 * SACC_L;
    if (warp < NCW) {
        for (int i = lane; i < 2 * SACC_L; i += 32) pw[i] = 0;
        __syncwarp();
#if PBCG_WIN_DRAIN
        long long *win = ring + (size_t)(NCW + 1) * 2 * SACC_L + (size_t)warp * WIN_WORDS;  // behind every warp's words
        d0.warp_merge_win(pw, win);
        d1.warp_merge_win(pw + SACC_L, win);
#else
        d0.warp_merge_priv(pw);
        d1.warp_merge_priv(pw + SACC_L);
#endif
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < 2 * 2 * SACC_L; idx += blockDim.x) {  // (group, accumulator, word)
        const int g = idx / (2 * SACC_L), k = (idx / SACC_L) & 1, i = idx % SACC_L;
        const int d = dot(g, k);
        if (d < 0) continue;
        long long t = 0;
#pragma unroll 4
        for (int wg = 0; wg < W; ++wg) t += ring[((size_t)(g * W + wg) * 2 + k) * SACC_L + i];
        if (t) S.w[d][i] += (unsigned long long)t;
    }
    __syncthreads();
}

// ---------------------------------------------------------------------------
// K2 (Alg. 2 l.70-74) + phase-A dots.  The consumer warps form two dot
// groups of W warps that see the same tiles: group 0 owns (q,y), (y,y) and
// stores p,s,z,q,y; group 1 recomputes s,z (8 FMAs) and owns (r0,s), (r0,z).
// Splitting the dots halves the accumulator registers per thread, which buys
// twice the warps (the ExBLAS cascades are latency-bound chains of DADDs).
// ---------------------------------------------------------------------------
template <class Acc>
struct K2Op {
    Acc d0, d1;
    double be, nom, nal;
    bool first;
    __device__ __forceinline__ void sz(double w, double t, double v, double &s, double &z) const {
        if (first) {  // beta_{-1} = 0: exact copies (R-3)
            s = w; z = t;
        } else {
            s = __fma_rn(be, __fma_rn(nom, z, s), w);  // s := w + beta (s - omega z)   l.71
            z = __fma_rn(be, __fma_rn(nom, v, z), t);  // z := t + beta (z - omega v)   l.72
        }
    }
    // group 0: p,s,z,q,y and the products of (q,y), (y,y)
    __device__ __forceinline__ void row0(unsigned &flags, double r, double w, double t, double v, double &p,
                                         double &s, double &z, double &q, double &y, Prod &P0, Prod &P1) {
        p = first ? r : __fma_rn(be, __fma_rn(nom, s, p), r);  // p := r + beta (p - omega s)   l.70
        sz(w, t, v, s, z);
        q = __fma_rn(nal, s, r);  // q := r - alpha s   l.73
        y = __fma_rn(nal, z, w);  // y := w - alpha z   l.74
        const bool zy = is_zero(y);
        P0 = d0.prep(q, y, is_zero(q) | zy, flags);
        P1 = d1.prep(y, y, zy, flags);
    }
    // group 1: s,z and the products of (r0,s), (r0,z)
    __device__ __forceinline__ void row1(unsigned &flags, double rh, double w, double t, double v, double s, double z,
                                         Prod &P0, Prod &P1) {
        sz(w, t, v, s, z);
        const bool zr = is_zero(rh);
        P0 = d0.prep(rh, s, zr | is_zero(s), flags);
        P1 = d1.prep(rh, z, zr | is_zero(z), flags);
    }
};

// EXACT = false: plain fp64 dots (PlainAcc, dot_mode PBCG_DOT_PLAIN).
// PIPE: the pipelined block Jacobi (R-25) also writes z_hat = M^-1 z (its own
// instantiation: the extra loads and FMAs would push the plain kernel past
// its register budget)
template <int NH, int NL, int W, int PPT, int STAGES, int NHE, bool EXACT = true, bool PIPE = false>
__global__ void __launch_bounds__((2 * W + 1) * 32, 1) k2_stream(K2Args a) {
    using Acc = typename std::conditional<EXACT, ExAccT<NH, NL, NHE>, PlainAcc>::type;
    constexpr int NV = 8;  // r, rh, w, t | p, s, z, v
    constexpr int NCW = 2 * W;
    constexpr int T = TileGeo<W, PPT>::T;
    static_assert(drain_ring_words(NCW + 1) <= (size_t)STAGES * NV * T, "the drain's scratch must fit in the ring");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *buf = (double *)smem_raw;
    uint64_t *full = (uint64_t *)(buf + (size_t)STAGES * NV * T);
    uint64_t *empty = full + STAGES;
    __shared__ CtaSacc<4> S;
    Scalars *sc = a.sc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PBCG_TL(0, 0);
#ifdef PBCG_TIMELINE
    if (threadIdx.x == 0 && blockIdx.x < 256) {
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        g_tl[0][blockIdx.x][7] = smid;
    }
#endif
    cta_sacc_zero<4>(S);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NCW); }
        mbar_fence_init();
    }
    __syncthreads();
    bool run;
    if (warp == NCW) {  // producer: r, r^, w, p, s, z, v stream out before the PDL wait; t (the SpMV's) after
        bool ok = true;
        if (lane == 0) {
            const bool first0 = (sc->it == 0);  // written by the previous finalize: complete (event dependency)
            const double *src[NV] = {a.r, a.rh, a.w, a.t, a.p, a.s, a.z, a.v};
            ok = produce_gated<NV, T, STAGES, PBCG_K2_EFM, PBCG_K2_ELM>(src, first0 ? 4 : 8, 3, a.n, buf, full, empty, [&]() {
                pdl_sync();
                return !sc->done;
            });
        }
        run = __shfl_sync(0xFFFFFFFFu, ok, 0);
    } else {
        pdl_sync();  // the previous kernel's vectors and scalars are complete from here on
        run = !sc->done;
    }
    if (!run) return;  // the whole CTA: done is the same value for every thread
    PBCG_TS(0);
    PBCG_TL(0, 1);
    const bool first = (sc->it == 0);
    const int64_t n = a.n;
    unsigned flags = 0;
    [[maybe_unused]] const uint64_t stpol = PBCG_K2_STM ? l2_policy_evict_first() : 0ull;
    K2Op<Acc> R;
    R.first = first;
    R.be = sc->beta;
    R.nom = -sc->omega;
    R.nal = -sc->alpha;
    R.d0.zero();
    R.d1.zero();
    const int g = warp / W, wg = warp % W;
    if constexpr (!EXACT) {  // per-warp slot of the plain sums (producer warp: none)
        R.d0.slot = warp < NCW ? wg : -1;
        R.d1.slot = warp < NCW ? wg : -1;
    }
    unsigned long long *s0 = S.w[2 * g], *s1 = S.w[2 * g + 1];
    if (warp < NCW) {  // consumers (the producer warp joins again for the merge)
        const int64_t ntiles = (n + T - 1) / T;
        int st = 0;
        uint32_t ph = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            mbar_wait(&full[st], ph);
            if (tile == blockIdx.x) PBCG_TL(0, 2);
            const int64_t r0 = tile * T;
            const int rows = (int)min((int64_t)T, n - r0);
            const int rows_even = rows & ~1;
            const double *B = buf + (size_t)st * NV * T;
            const double2 *B2 = (const double2 *)B;
            constexpr int TP = T / 2;  // double2 per vector slice
#pragma unroll
            for (int u = 0; u < PPT; ++u) {
                const int j = u * W * 32 + wg * 32 + lane;  // pair index in the tile
                const int jw = u * W * 32 + wg * 32 + 31;
                const int64_t gp = (r0 >> 1) + j;          // global pair index
                if (2 * jw + 1 < rows_even) {              // whole warp valid
                    const double2 w = B2[2 * TP + j], t = B2[3 * TP + j];
                    double2 ss, z, v;
                    if (!first) { ss = B2[5 * TP + j]; z = B2[6 * TP + j]; v = B2[7 * TP + j]; }
                    Prod P[4];
                    if (g == 0) {
                        const double2 r = B2[0 * TP + j];
                        double2 p, q, y;
                        if (!first) p = B2[4 * TP + j];
                        R.row0(flags, r.x, w.x, t.x, v.x, p.x, ss.x, z.x, q.x, y.x, P[0], P[1]);
                        R.row0(flags, r.y, w.y, t.y, v.y, p.y, ss.y, z.y, q.y, y.y, P[2], P[3]);
                        st_v2<PBCG_K2_STM, 0>(a.p, gp, p, stpol); st_v2<PBCG_K2_STM, 1>(a.s, gp, ss, stpol);
                        st_v2<PBCG_K2_STM, 2>(a.z, gp, z, stpol); st_v2<PBCG_K2_STM, 3>(a.q, gp, q, stpol);
                        st_v2<PBCG_K2_STM, 4>(a.y, gp, y, stpol);
                        if constexpr (PIPE) ((double2 *)a.zh)[gp] = bj_pair(a.minv, gp, z.x, z.y);  // z_hat = M^-1 z (R-25)
                    } else {
                        const double2 rh = B2[1 * TP + j];
                        R.row1(flags, rh.x, w.x, t.x, v.x, ss.x, z.x, P[0], P[1]);
                        R.row1(flags, rh.y, w.y, t.y, v.y, ss.y, z.y, P[2], P[3]);
                    }
                    cascade_batch<4, true, PBCG_VSPLIT_K2(NL)>(R.d0, R.d1, P, s0, s1);
                } else {
                    [[maybe_unused]] double zz[2] = {0.0, 0.0};  // this pair's z (pipelined block Jacobi)
                    for (int h = 0; h < 2; ++h) {
                        const int lr = 2 * j + h;  // local row
                        if (lr >= rows) break;
                        const int64_t gi = r0 + lr;
                        const bool m = lr < rows_even;
                        const double w = m ? B[2 * T + lr] : a.w[gi], t = m ? B[3 * T + lr] : a.t[gi];
                        double ss = 0, z = 0, v = 0;
                        Prod P0, P1;
                        if (!first) {
                            ss = m ? B[5 * T + lr] : a.s[gi]; z = m ? B[6 * T + lr] : a.z[gi];
                            v = m ? B[7 * T + lr] : a.v[gi];
                        }
                        if (g == 0) {
                            const double r = m ? B[0 * T + lr] : a.r[gi];
                            double p = 0, q, y;
                            if (!first) p = m ? B[4 * T + lr] : a.p[gi];
                            R.row0(flags, r, w, t, v, p, ss, z, q, y, P0, P1);
                            a.p[gi] = p; a.s[gi] = ss; a.z[gi] = z; a.q[gi] = q; a.y[gi] = y;
                            if constexpr (PIPE) zz[h] = z;
                        } else {
                            R.row1(flags, m ? B[1 * T + lr] : a.rh[gi], w, t, v, ss, z, P0, P1);
                        }
                        cascade_one(R.d0, P0, s0);
                        cascade_one(R.d1, P1, s1);
                    }
                    if (PIPE && g == 0 && 2 * j < rows) {  // z_hat of the pair; an odd last row is the 1x1 tail block
                        const int64_t m0 = (r0 >> 1) + j;
                        if (2 * j + 1 < rows) ((double2 *)a.zh)[m0] = bj_pair(a.minv, m0, zz[0], zz[1]);
                        else a.zh[2 * m0] = __dmul_rn(a.minv[4 * m0], zz[0]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == STAGES) { st = 0; ph ^= 1u; }
        }
    }
    PBCG_TS(1);
    PBCG_TL(0, 3);
    __syncwarp();
#ifndef PBCG_OLD_DRAIN
    if constexpr (EXACT) {  // dots 2g, 2g+1 of group g
        drain_private<4, NCW, W>(S, R.d0, R.d1, (long long *)buf, [](int g, int k) { return 2 * g + k; });
    } else
#endif
    {
        R.d0.warp_merge(s0);
        R.d1.warp_merge(s1);
    }
    PBCG_TS(2);
    PBCG_TL(0, 4);
    if constexpr (EXACT) {
        if (sc->range_mode == 0) {  // full range (R-24): a flagged CTA corrects its products
            if (flags) atomicOr(&S.flags, flags);
            flags = 0;
            __syncthreads();  // the ring is drained (its memory is the scratch); this CTA's q, y, s, z stores are visible
            if (S.flags & FLAG_RANGE)
                cta_full_range_nd<4>(S, (unsigned long long *)buf, a.gacc + xs_off(4),
                    [&](auto f) {
                        for (int64_t tile = blockIdx.x; tile * T < n; tile += gridDim.x) {
                            const int64_t e = min(n, tile * T + T);
                            for (int64_t i = tile * T + threadIdx.x; i < e; i += blockDim.x) f(i);
                        }
                    },
                    [&](int d, int64_t i, double &x, double &y) {  // (q,y), (y,y), (r0,s), (r0,z)
                        const double yi = a.y[i];
                        x = d == 0 ? a.q[i] : d == 1 ? yi : a.rh[i];
                        y = d <= 1 ? yi : d == 2 ? a.s[i] : a.z[i];
                    });
        }
        const bool last = cta_sacc_publish<4>(S, flags, a.gacc, a.ticket);
        PBCG_TS(3);
        PBCG_TL(0, 5);
        if (last) {
            last_cta_finish<4>(S, a.gacc, a.ticket, PH_A, a.finalize, sc, a.hist, nullptr, nullptr);
            PBCG_TS(4);
        }
    } else {
        plain_publish<4, W>(S, a.part);
    }
}

// ---------------------------------------------------------------------------
// K3 (Alg. 2 l.77-79) + phase-B dots.  Group 0: x, r' and (r0,r'), (r',r');
// group 1: w' and (r0,w').
// ---------------------------------------------------------------------------
template <class Acc>
struct K3Op {
    Acc d0, d1;
    double al, om, nal, nom;
    // group 0: x, r' and the products of (r0,r'), (r',r')
    __device__ __forceinline__ void row0(unsigned &flags, double rh, double p, double q, double y, double &x, double &r,
                                         Prod &P0, Prod &P1) {
        x = __fma_rn(om, q, __fma_rn(al, p, x));  // x := x + alpha p + omega q      l.77
        r = __fma_rn(nom, y, q);                  // r := q - omega y                l.78
        const bool zr = is_zero(r);
        P0 = d0.prep(rh, r, is_zero(rh) | zr, flags);
        P1 = d1.prep(r, r, zr, flags);
    }
    // group 1: w' and the product of (r0,w')
    __device__ __forceinline__ void row1(unsigned &flags, double rh, double y, double t, double v, double &w,
                                         Prod &P0) {
        w = __fma_rn(nom, __fma_rn(nal, v, t), y);  // w := y - omega (t - alpha v)    l.79
        P0 = d0.prep(rh, w, is_zero(rh) | is_zero(w), flags);
    }
};

template <int NH, int NL, int W, int PPT, int STAGES, int NHE, bool EXACT = true, bool PIPE = false>
__global__ void __launch_bounds__((2 * W + 1) * 32, 1) k3_stream(K3Args a) {
    using Acc = typename std::conditional<EXACT, ExAccT<NH, NL, NHE>, PlainAcc>::type;
    constexpr int NV = 7;  // rh, p, q, y, t, v, x
    constexpr int NCW = 2 * W;
    constexpr int T = TileGeo<W, PPT>::T;
    static_assert(drain_ring_words(NCW + 1) <= (size_t)STAGES * NV * T, "the drain's scratch must fit in the ring");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *buf = (double *)smem_raw;
    uint64_t *full = (uint64_t *)(buf + (size_t)STAGES * NV * T);
    uint64_t *empty = full + STAGES;
    __shared__ CtaSacc<3> S;
    Scalars *sc = a.sc;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PBCG_TL(2, 0);
    cta_sacc_zero<3>(S);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NCW); }
        mbar_fence_init();
    }
    __syncthreads();
    bool run;
    if (warp == NCW) {  // producer: everything but v (the SpMV's) streams out before the PDL wait
        bool ok = true;
        if (lane == 0) {
            const double *src[NV] = {a.rh, a.p, a.q, a.y, a.t, a.v, a.x};
            ok = produce_gated<NV, T, STAGES, PBCG_K3_EFM, PBCG_K3_ELM>(src, NV, 5, a.n, buf, full, empty, [&]() {
                pdl_sync();
                return !sc->done;
            });
        }
        run = __shfl_sync(0xFFFFFFFFu, ok, 0);
    } else {
        pdl_sync();
        run = !sc->done;
    }
    if (!run) return;
    PBCG_TL(2, 1);
    const int64_t n = a.n;
    unsigned flags = 0;
    [[maybe_unused]] const uint64_t stpol = PBCG_K3_STM ? l2_policy_evict_first() : 0ull;
    K3Op<Acc> R;
    R.al = sc->alpha;
    R.om = sc->omega;
    R.nal = -R.al;
    R.nom = -R.om;
    R.d0.zero();
    R.d1.zero();
    const int g = warp / W, wg = warp % W;
    if constexpr (!EXACT) {  // per-warp slot of the plain sums; group 1 has one dot, the producer none
        R.d0.slot = warp < NCW ? wg : -1;
        R.d1.slot = (warp < NCW && g == 0) ? wg : -1;
    }
    // dot slots: (r0,r') -> 0, (r0,w') -> 1, (r',r') -> 2
    unsigned long long *s0 = S.w[g == 0 ? 0 : 1], *s1 = S.w[2];
    if (warp < NCW) {  // consumers (the producer warp joins again for the merge)
        const int64_t ntiles = (n + T - 1) / T;
        int st = 0;
        uint32_t ph = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            mbar_wait(&full[st], ph);
            if (tile == blockIdx.x) PBCG_TL(2, 2);
            const int64_t r0 = tile * T;
            const int rows = (int)min((int64_t)T, n - r0);
            const int rows_even = rows & ~1;
            const double *B = buf + (size_t)st * NV * T;
            const double2 *B2 = (const double2 *)B;
            constexpr int TP = T / 2;
#pragma unroll
            for (int u = 0; u < PPT; ++u) {
                const int j = u * W * 32 + wg * 32 + lane;
                const int jw = u * W * 32 + wg * 32 + 31;
                const int64_t gp = (r0 >> 1) + j;
                if (2 * jw + 1 < rows_even) {
                    const double2 rh = B2[0 * TP + j], y = B2[3 * TP + j];
                    if (g == 0) {
                        const double2 p = B2[1 * TP + j], q = B2[2 * TP + j];
                        double2 x = B2[6 * TP + j], r;
                        Prod P[4];
                        R.row0(flags, rh.x, p.x, q.x, y.x, x.x, r.x, P[0], P[1]);
                        R.row0(flags, rh.y, p.y, q.y, y.y, x.y, r.y, P[2], P[3]);
                        st_v2<PBCG_K3_STM, 0>(a.x, gp, x, stpol); st_v2<PBCG_K3_STM, 1>(a.r, gp, r, stpol);
                        cascade_batch<4, true, PBCG_VSPLIT_K3(NL)>(R.d0, R.d1, P, s0, s1);
                    } else {
                        const double2 t = B2[4 * TP + j], v = B2[5 * TP + j];
                        double2 w;
                        Prod P[2];
                        R.row1(flags, rh.x, y.x, t.x, v.x, w.x, P[0]);
                        R.row1(flags, rh.y, y.y, t.y, v.y, w.y, P[1]);
                        st_v2<PBCG_K3_STM, 2>(a.w, gp, w, stpol);
                        if constexpr (PIPE) ((double2 *)a.wh)[gp] = bj_pair(a.minv, gp, w.x, w.y);  // w_hat = M^-1 w (R-25)
                        cascade_batch<2, false>(R.d0, R.d1, P, s0, s1);
                    }
                } else {
                    [[maybe_unused]] double ww[2] = {0.0, 0.0};  // this pair's w (pipelined block Jacobi)
                    for (int h = 0; h < 2; ++h) {
                        const int lr = 2 * j + h;
                        if (lr >= rows) break;
                        const int64_t gi = r0 + lr;
                        const bool m = lr < rows_even;
                        const double rh = m ? B[0 * T + lr] : a.rh[gi], y = m ? B[3 * T + lr] : a.y[gi];
                        if (g == 0) {
                            double x = m ? B[6 * T + lr] : a.x[gi], r;
                            Prod P0, P1;
                            R.row0(flags, rh, m ? B[1 * T + lr] : a.p[gi], m ? B[2 * T + lr] : a.q[gi], y, x, r, P0, P1);
                            a.x[gi] = x; a.r[gi] = r;
                            cascade_one(R.d0, P0, s0);
                            cascade_one(R.d1, P1, s1);
                        } else {
                            double w;
                            Prod P0;
                            R.row1(flags, rh, y, m ? B[4 * T + lr] : a.t[gi], m ? B[5 * T + lr] : a.v[gi], w, P0);
                            a.w[gi] = w;
                            if constexpr (PIPE) ww[h] = w;
                            cascade_one(R.d0, P0, s0);
                        }
                    }
                    if (PIPE && g == 1 && 2 * j < rows) {
                        const int64_t m0 = (r0 >> 1) + j;
                        if (2 * j + 1 < rows) ((double2 *)a.wh)[m0] = bj_pair(a.minv, m0, ww[0], ww[1]);
                        else a.wh[2 * m0] = __dmul_rn(a.minv[4 * m0], ww[0]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[st]);
            if (++st == STAGES) { st = 0; ph ^= 1u; }
        }
    }
    PBCG_TL(2, 3);
    __syncwarp();
#ifndef PBCG_OLD_DRAIN
    if constexpr (EXACT) {  // group 0: (r0,r') -> 0, (r',r') -> 2; group 1: (r0,w') -> 1
        drain_private<3, NCW, W>(S, R.d0, R.d1, (long long *)buf,
                                 [](int g, int k) { return g == 0 ? (k == 0 ? 0 : 2) : (k == 0 ? 1 : -1); });
    } else
#endif
    {
        R.d0.warp_merge(s0);
        R.d1.warp_merge(s1);
    }
    PBCG_TL(2, 4);
    if constexpr (EXACT) {
        if (sc->range_mode == 0) {  // full range (R-24): a flagged CTA corrects its products
            if (flags) atomicOr(&S.flags, flags);
            flags = 0;
            __syncthreads();
            if (S.flags & FLAG_RANGE)
                cta_full_range_nd<3>(S, (unsigned long long *)buf, a.gacc + xs_off(3),
                    [&](auto f) {
                        for (int64_t tile = blockIdx.x; tile * T < n; tile += gridDim.x) {
                            const int64_t e = min(n, tile * T + T);
                            for (int64_t i = tile * T + threadIdx.x; i < e; i += blockDim.x) f(i);
                        }
                    },
                    [&](int d, int64_t i, double &x, double &y) {  // (r0,r'), (r0,w'), (r',r')
                        const double ri = a.r[i];
                        x = d <= 1 ? a.rh[i] : ri;
                        y = d == 1 ? a.w[i] : ri;
                    });
        }
        const bool last = cta_sacc_publish<3>(S, flags, a.gacc, a.ticket);
        PBCG_TL(2, 5);
        if (last) last_cta_finish<3>(S, a.gacc, a.ticket, PH_B, a.finalize, sc, a.hist, nullptr, nullptr);
    } else {
        plain_publish<3, W>(S, a.part);
    }
}

// ---------------------------------------------------------------------------
#ifndef PBCG_XD_PRIV_DRAIN
#define PBCG_XD_PRIV_DRAIN 1  // 2^26: WELL 6,517 -> 6,591 GB/s, ILL 4,117 -> 4,172; 2^22 ILL 1,861 -> 1,985 (tools/exdot_bench.py)
#endif
// Standalone EXDOT (one dot, x and y 16-byte aligned)
// ---------------------------------------------------------------------------
// ND = 2: the dots (x,y) and (y,y) over the same two streams (Alg. 1's
// (q,y),(y,y) and (r0,r),(r,r) phases); products alternate between the two
// accumulators inside one batched cascade.
template <int NH, int NL, int NCW, int PPT, int STAGES, int ND = 1>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) exdot_stream(MultiDotArgs a) {
    static_assert(ND == 1 || ND == 2, "ND is 1 or 2");
    constexpr int NV = 2;
    constexpr int T = TileGeo<NCW, PPT>::T;
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *buf = (double *)smem_raw;
    uint64_t *full = (uint64_t *)(buf + (size_t)STAGES * NV * T);
    uint64_t *empty = full + STAGES;
    __shared__ CtaSacc<ND> S;
    if (a.sc && a.sc->done && a.phase != PH_TRUE) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    cta_sacc_zero<ND>(S);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], NCW); }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t n = a.n;
    unsigned flags = 0;
    ExAccT<NH, NL> acc, acc2;
    acc.zero();
    acc2.zero();
    unsigned long long *s1 = S.w[ND - 1];
    if (warp == NCW) {
        if (lane == 0) {
            const double *src[NV] = {a.x[0], a.y[0]};
            produce<NV, T, STAGES>(src, NV, n, buf, full, empty);
        }
    } else {
        const int64_t ntiles = (n + T - 1) / T;
        int s = 0;
        uint32_t ph = 0;
        for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
            mbar_wait(&full[s], ph);
            const int64_t r0 = tile * T;
            const int rows = (int)min((int64_t)T, n - r0);
            const int rows_even = rows & ~1;
            const double *B = buf + (size_t)s * NV * T;
            const int jw0 = warp * 32 + 31;
            if (2 * ((PPT - 1) * NCW * 32 + jw0) + 1 < rows_even) {  // whole tile slice valid
                double2 xv[PPT], yv[PPT];
#pragma unroll
                for (int u = 0; u < PPT; ++u) {
                    const int j = u * NCW * 32 + warp * 32 + lane;
                    xv[u] = ((const double2 *)B)[j];
                    yv[u] = ((const double2 *)(B + T))[j];
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);  // operands are in registers: free the slot early
                if (ND == 1) {
#pragma unroll
                    for (int u = 0; u < PPT; u += 2) {
                        Prod P[4];
#pragma unroll
                        for (int h = 0; h < 2 && u + h < PPT; ++h) {
                            P[2 * h] = acc.prep(xv[u + h].x, yv[u + h].x, is_zero(xv[u + h].x) | is_zero(yv[u + h].x), flags);
                            P[2 * h + 1] = acc.prep(xv[u + h].y, yv[u + h].y, is_zero(xv[u + h].y) | is_zero(yv[u + h].y), flags);
                        }
                        cascade_batch<4, false>(acc, acc, P, S.w[0], S.w[0]);
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < PPT; ++u) {
                        Prod P[4];  // (x,y) -> acc, (y,y) -> acc2, alternating
                        const bool zy0 = is_zero(yv[u].x), zy1 = is_zero(yv[u].y);
                        P[0] = acc.prep(xv[u].x, yv[u].x, is_zero(xv[u].x) | zy0, flags);
                        P[1] = acc2.prep(yv[u].x, yv[u].x, zy0, flags);
                        P[2] = acc.prep(xv[u].y, yv[u].y, is_zero(xv[u].y) | zy1, flags);
                        P[3] = acc2.prep(yv[u].y, yv[u].y, zy1, flags);
                        cascade_batch<4, true>(acc, acc2, P, S.w[0], s1);
                    }
                }
            } else {
#pragma unroll
                for (int u = 0; u < PPT; ++u) {
                    const int j = u * NCW * 32 + warp * 32 + lane;
                    for (int h = 0; h < 2; ++h) {
                        const int lr = 2 * j + h;
                        if (lr >= rows) break;
                        const bool m = lr < rows_even;
                        const double xv = m ? B[lr] : a.x[0][r0 + lr], yv = m ? B[T + lr] : a.y[0][r0 + lr];
                        cascade_one(acc, acc.prep(xv, yv, is_zero(xv) | is_zero(yv), flags), S.w[0]);
                        if (ND == 2) cascade_one(acc2, acc2.prep(yv, yv, is_zero(yv), flags), s1);
                    }
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[s]);
            }
            if (++s == STAGES) { s = 0; ph ^= 1u; }
        }
    }
    __syncwarp();
#if PBCG_XD_PRIV_DRAIN
    // one dot group of NCW warps: accumulator k -> dot k (acc2 stays zero when ND = 1)
    static_assert(drain_ring_words(NCW + 1) <= (size_t)STAGES * NV * T, "the drain's scratch must fit in the ring");
    drain_private<ND, NCW, NCW>(S, acc, acc2, (long long *)buf, [](int g, int k) { return (g == 0 && k < ND) ? k : -1; });
#else
    acc.warp_merge(S.w[0]);
    if (ND == 2) acc2.warp_merge(s1);
#endif
    if constexpr (ND == 2) {
        if (phase_full_range(a.phase, a.sc)) {  // Algorithm 2's init with x0 = 0 (PH_INIT0): R-24 as in K2/K3
            if (flags) atomicOr(&S.flags, flags);
            flags = 0;
            __syncthreads();  // the ring is drained: its memory is the scratch
            if (S.flags & FLAG_RANGE)
                cta_full_range_nd<2>(S, (unsigned long long *)buf, a.gacc + xs_off(2),
                    [&](auto f) {
                        for (int64_t tile = blockIdx.x; tile * T < n; tile += gridDim.x) {
                            const int64_t e = min(n, tile * T + T);
                            for (int64_t i = tile * T + threadIdx.x; i < e; i += blockDim.x) f(i);
                        }
                    },
                    [&](int d, int64_t i, double &x, double &y) {  // (x,y), (y,y)
                        y = a.y[0][i];
                        x = d == 0 ? a.x[0][i] : y;
                    });
        }
    }
    if constexpr (ND == 1) {
        if (a.phase == PH_EXDOT) {  // standalone dot (single GPU or a rank's slice): a flagged CTA corrects its products (NEXT-4)
            if (flags) atomicOr(&S.flags, flags);
            flags = 0;
            __syncthreads();  // the ring is drained: its memory is the scratch
            if (S.flags)
                cta_full_range<NCW + 1>(S, (unsigned long long *)buf, a.gacc, a.x[0], a.y[0], [&](auto f) {
                    for (int64_t tile = blockIdx.x; tile * T < n; tile += gridDim.x) {
                        const int64_t e = min(n, tile * T + T);
                        for (int64_t i = tile * T + threadIdx.x; i < e; i += blockDim.x) f(i);
                    }
                });
        }
    }
    if (cta_sacc_publish<ND>(S, flags, a.gacc, a.ticket))
        last_cta_finish<ND>(S, a.gacc, a.ticket, a.phase, a.finalize, a.sc, a.hist, a.out, a.out_flags);
}

// ---------------------------------------------------------------------------
// SpMV (Alg. 2 l.75 v = A z, l.80 t = A w) for matrices whose rows hold <= 8
// nonzeros (the stencil configs), from the packed sliced-ELL format SELL-P:
// chunk c = SPS consecutive 32-row slices stored as ONE contiguous blob
//   header: vo[SPS+1] (int32, value offset of each slice in the blob's value
//           area), xo[SPS+1] (int32, offset of each slice's explicit column
//           ids), len[SPS*32] (uint8 row lengths), rec[SPS*16] (slot records:
//           uniform pos-relative column per slot + mask, SellMat::slot_rec)
//   values: slot-major, 32 per slot, widths of the slices
//   explicit column ids: pos-relative, 32 per non-uniform slot
// so the producer lane moves a chunk with one bulk copy (the TMA engine's
// per-copy cost is what limits small-copy streaming).  All consumer warps read
// each stage: warp j folds slice j -- x gathered through L1/L2 (x is read
// from HBM once: banded matrix), the row's ordered fma chain (R-6) -- and
// stores y.  Column ids of uniform slots are never stored.
// ---------------------------------------------------------------------------
template <int SPS>
struct SellPGeo {
    static constexpr int HO1 = ((SPS + 1) * 4 + 15) / 16 * 16;       // xo[]
    static constexpr int HO2 = 2 * HO1;                              // len[] (uint8)
    static constexpr int HO3 = HO2 + SPS * 32;                       // rec[]
    static constexpr int H = (HO3 + SPS * SELL_RS * 4 + 127) / 128 * 128;  // values start
    static constexpr int MAXBLOB = H + SPS * 32 * 8 * (8 + 4);       // width <= 8, all slots explicit
};

// per slice: number of explicit (non-uniform) slots among its width
__global__ void sellp_count_kernel(int64_t nslices, const int64_t *slice_off, const int32_t *slot_rec, uint8_t *nexp) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslices; s += (int64_t)gridDim.x * blockDim.x) {
        const int W = (int)((slice_off[s + 1] - slice_off[s]) >> 5);
        const uint32_t m = slot_rec ? (uint32_t)slot_rec[s * SELL_RS + SELL_MASK] : 0u;
        nexp[s] = (uint8_t)__popc(~m & ((1u << W) - 1u));
    }
}

// one warp per slice: scatter its header entries, values and explicit column
// ids into its chunk's blob (blob zeroed beforehand: lengths past n stay 0)
template <int SPS>
__global__ void sellp_fill_kernel(int64_t n, int64_t nslices, SellMat A, const uint8_t *nexp, const int64_t *blob_off,
                                  unsigned char *blob) {
    using Geo = SellPGeo<SPS>;
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += nw) {
        const int64_t c = s / SPS;
        const int j = (int)(s % SPS);
        unsigned char *bb = blob + blob_off[c];
        const int64_t so = A.slice_off[s], so0 = A.slice_off[c * SPS];
        const int W = (int)((A.slice_off[s + 1] - so) >> 5);
        const int vo = (int)(so - so0);
        int xo = (lane < j) ? nexp[c * SPS + lane] : 0;
        xo = 32 * __reduce_add_sync(0xFFFFFFFFu, xo);
        const uint32_t m = A.slot_rec ? (uint32_t)A.slot_rec[s * SELL_RS + SELL_MASK] : 0u;
        const int64_t nvc = A.slice_off[min((c + 1) * SPS, nslices)] - so0;  // values of the chunk
        if (lane == 0) {
            ((int32_t *)bb)[j] = vo;
            ((int32_t *)(bb + Geo::HO1))[j] = xo;
            if (j == 0) ((int32_t *)bb)[SPS] = (int32_t)nvc;
        }
        const int64_t pos = s * 32 + lane;
        bb[Geo::HO2 + j * 32 + lane] = (uint8_t)(pos < n ? A.row_len[pos] : 0);
        if (lane < SELL_RS)
            ((int32_t *)(bb + Geo::HO3))[j * SELL_RS + lane] = A.slot_rec ? A.slot_rec[s * SELL_RS + lane] : 0;
        double *bv = (double *)(bb + Geo::H);
        int32_t *bx = (int32_t *)(bb + Geo::H + 8 * nvc);
        int q = 0;
        for (int k = 0; k < W; ++k) {
            bv[vo + 32 * k + lane] = A.val[so + 32 * k + lane];
            if (!((m >> k) & 1u)) bx[xo + 32 * (q++) + lane] = A.col[so + 32 * k + lane];
        }
    }
}

// Producer warp of the SELL-P kernels: the blob extents of 32 chunks per
// batch are loaded one per lane (the next batch in flight during this one),
// lane 0 moves each chunk of this CTA with ONE bulk copy into the ring.
// `gate` (all lanes; returns false to abort) runs after the first `prefill`
// chunks are issued: the SpMV's matrix stream is static, so the producer
// starts it before waiting on the previous kernel (PDL); on abort it drains
// the copies it issued, so none is in flight when the CTA exits.
template <class Gate>
__device__ __forceinline__ void sellp_produce(int64_t cbeg, int64_t nchunks, const unsigned char *blob,
                                              const int64_t *blob_off,
                                              unsigned char *smem, int STAGE, int STAGES, uint64_t *full,
                                              uint64_t *empty, int prefill, Gate gate) {
    const int lane = threadIdx.x & 31;
    auto extents = [&](int64_t k, int64_t &c, int64_t &o0, int64_t &o1) {
        c = cbeg + blockIdx.x + k * gridDim.x;
        o0 = o1 = 0;
        if (c < nchunks) {
            o0 = __ldg(&blob_off[c]);
            o1 = __ldg(&blob_off[c + 1]);
        }
    };
    int issued = 0;
    bool gated = false;
    const uint64_t pol = l2_policy_evict_first();
    auto pass_gate = [&]() {
        gated = true;
        if (gate()) return true;
        if (lane == 0)
            for (int s = 0; s < issued; ++s) mbar_wait(&full[s], 0u);  // first pass only: issued <= STAGES
        __syncwarp();
        return false;
    };
    int64_t cc, c0, c1, nc, n0, n1;
    extents(lane, cc, c0, c1);
    int st = 0;
    uint32_t ph = 0;
    for (int64_t kb = 0;; kb += 32) {
        if (__shfl_sync(0xFFFFFFFFu, cc, 0) >= nchunks) break;
        extents(kb + 32 + lane, nc, n0, n1);
        for (int l = 0; l < 32; ++l) {
            const int64_t c = __shfl_sync(0xFFFFFFFFu, cc, l);
            if (c >= nchunks) break;
            if (!gated && issued == prefill && !pass_gate()) return;
            const int64_t o0 = __shfl_sync(0xFFFFFFFFu, c0, l), o1 = __shfl_sync(0xFFFFFFFFu, c1, l);
            if (lane == 0) {
                mbar_wait(&empty[st], ph ^ 1u);
                mbar_expect_tx(&full[st], (uint32_t)(o1 - o0));
                bulk_g2s_stream(smem + (size_t)st * STAGE, blob + o0, (uint32_t)(o1 - o0), &full[st], pol);
            }
            ++issued;
            if (++st == STAGES) {
                st = 0;
                ph ^= 1u;
            }
            __syncwarp();
        }
        cc = nc;
        c0 = n0;
        c1 = n1;
    }
    if (!gated) pass_gate();
}

// STAGE (bytes, multiple of 128) = the largest chunk blob of this matrix,
// STAGES = as many as fit in shared memory (set at setup).
template <int MODE, int SPS, int RPW>
__global__ void __launch_bounds__((SPS / RPW + 1) * 32, 1)
    spmv_sellp_kernel(int64_t n, int64_t nslices, const unsigned char *__restrict__ blob,
                      const int64_t *__restrict__ blob_off, const int32_t *__restrict__ perm,
                      const double *__restrict__ x, double *__restrict__ y, const double *__restrict__ b,
                      double *__restrict__ y2, const Scalars *sc, int STAGE, int STAGES, int64_t cbeg, int64_t cend) {
    // chunks [cbeg, cend) (interior / boundary split under multi-rank halo overlap)
    using Geo = SellPGeo<SPS>;
    constexpr int NCW = SPS / RPW;  // consumer warps
    static_assert(SPS % RPW == 0, "SPS must be a multiple of RPW");
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *full = (uint64_t *)(smem_raw + (size_t)STAGES * STAGE);
    uint64_t *empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PBCG_TL(1, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    const int64_t nchunks = cend;
    if (warp == NCW) {  // producer warp: the first STAGES chunks go out before the PDL wait
        sellp_produce(cbeg, nchunks, blob, blob_off, smem_raw, STAGE, STAGES, full, empty, STAGES, [&]() {
            pdl_sync();
            return !(sc && sc->done);
        });
        return;
    }
    pdl_sync();
    if (sc && sc->done) return;
    PBCG_TL(1, 1);
    // gathers of a chunk's RPW slices of this warp (stage st)
    auto issue = [&](int64_t c, int st, int (&len)[RPW], double (&xv)[RPW][8]) {
        const unsigned char *sb = smem_raw + (size_t)st * STAGE;
        const int32_t *vo = (const int32_t *)sb;
        const int32_t *xo = (const int32_t *)(sb + Geo::HO1);
        const int32_t *rec = (const int32_t *)(sb + Geo::HO3);
        const int32_t *bx = (const int32_t *)((const double *)(sb + Geo::H) + vo[SPS]);  // explicit ids after values
#pragma unroll
        for (int u = 0; u < RPW; ++u) {
            const int j = warp * RPW + u;
            const int64_t s = c * SPS + j;
            len[u] = s < nslices ? sb[Geo::HO2 + j * 32 + lane] : 0;
            const int64_t pos = s * 32 + lane;
            const uint32_t m = (uint32_t)rec[j * SELL_RS + SELL_MASK];
            const int32_t *xs = bx + xo[j] + lane;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                // uniform slot: the record; else the next explicit column id
                if (k < len[u]) {
                    const bool uni = (m >> k) & 1u;
                    const int q = __popc(~m & ((1u << k) - 1u));
                    const int rel = uni ? rec[j * SELL_RS + k] : xs[32 * q];
                    xv[u][k] = __ldg(x + (pos + rel));
                }
            }
        }
    };
    // the folds and stores of those slices, then the stage goes back
    auto fold = [&](int64_t c, int st, const int (&len)[RPW], const double (&xv)[RPW][8]) {
        const unsigned char *sb = smem_raw + (size_t)st * STAGE;
        const int32_t *vo = (const int32_t *)sb;
        const double *bv = (const double *)(sb + Geo::H);
#pragma unroll
        for (int u = 0; u < RPW; ++u) {
            const int j = warp * RPW + u;
            const int64_t pos = (c * SPS + j) * 32 + lane;
            const double *vs = bv + vo[j] + lane;
            double acc = 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (k < len[u]) acc = __fma_rn(vs[32 * k], xv[u][k], acc);  // ordered chain, +0.0 start (R-6)
            if (pos < n) {
                const int64_t row = perm ? (int64_t)__ldg(&perm[pos]) : pos;
                if (MODE == SPMV_PLAIN) {
                    y[row] = acc;
                } else {
                    const double r = __dsub_rn(b[row], acc);  // r0 := b - A x0 (l.64)
                    y[row] = r;
                    if (y2) y2[row] = r;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
    };
    int st = 0;
    uint32_t ph = 0;
    int len[RPW];
    double xv[RPW][8];
    for (int64_t c = cbeg + blockIdx.x; c < nchunks; c += gridDim.x) {
        mbar_wait(&full[st], ph);
        if (c == cbeg + blockIdx.x) PBCG_TL(1, 2);
        issue(c, st, len, xv);
        fold(c, st, len, xv);
        if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
        }
    }
    PBCG_TL(1, 3);
}

// ---------------------------------------------------------------------------
// SELL-V: the TMA-streamed SpMV for long rows (irregular matrices, C4).
// The sliced ELL (C = 32, sigma-sorted) is cut into chunks of consecutive
// slices bounded by BYTES (a chunk is at most one ring stage), not by slice
// count, so a row may hold up to 255 nonzeros.  Within a slice the padding
// is dropped: slot k stores only the lanes whose row has a k-th nonzero, in
// lane order (a lane finds its entry by the popcount of the active lanes
// below it), so the stream is exactly the nonzeros.  Chunk blob:
//   int32 s0 (first slice), ns (slices), nval (entries), pad;
//   int32 vo[ns] (entry offset of each slice); uint8 len[ns][32];
//   (16-byte aligned) double val[nval]; int32 col[nval]  (pos-relative ids)
// One bulk copy moves a chunk.  Slice j of a chunk goes to consumer warp
// (rot + j) mod NCW, rot = the CTA's running slice count, so successive
// chunks fill successive warps and every warp walks the ring (waiting on
// each stage, arriving once per chunk): up to STAGES chunks of slices are
// folded concurrently.  Lane = row: its ordered fma chain (R-6) over the
// row's nonzeros, x gathered through L1/L2, UNR gathers in flight.
// ---------------------------------------------------------------------------
__host__ __device__ __forceinline__ int sellv_hdr_bytes(int ns) { return (16 + 36 * ns + 15) & ~15; }

// nonzeros per slice (the chunking runs on the host)
__global__ void sellv_count_kernel(int64_t n, int64_t nslices, const int32_t *row_len, int32_t *nnz_slice) {
    for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nslices; s += (int64_t)gridDim.x * blockDim.x) {
        int t = 0;
        for (int l = 0; l < 32; ++l) t += (s * 32 + l < n) ? row_len[s * 32 + l] : 0;
        nnz_slice[s] = t;
    }
}

// one warp per slice: header entries, values and column ids of the slice into
// its chunk (cs[c] = first slice of chunk c, vs[s] = entry offset of slice s
// inside its chunk; blob zeroed beforehand)
__global__ void sellv_fill_kernel(int64_t n, int64_t nslices, SellMat A, const int32_t *cs, const int32_t *vs,
                                  int64_t nchunks, const int64_t *blob_off, unsigned char *blob) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += nw) {
        int64_t lo = 0, hi = nchunks;  // chunk c with cs[c] <= s < cs[c + 1]
        while (hi - lo > 1) {
            const int64_t mid = (lo + hi) >> 1;
            if (cs[mid] <= s) lo = mid;
            else hi = mid;
        }
        const int64_t c = lo;
        const int ns = cs[c + 1] - cs[c];
        const int j = (int)(s - cs[c]);
        const int last = cs[c + 1] - 1;
        unsigned char *bb = blob + blob_off[c];
        int32_t *hd = (int32_t *)bb;
        const int64_t pos = s * 32 + lane;
        const int len = pos < n ? A.row_len[pos] : 0;
        const int W = (int)((A.slice_off[s + 1] - A.slice_off[s]) >> 5);
        const int vo = vs[s];
        // entries of the chunk = offset of its last slice + that slice's nonzeros
        int lastn = (last * 32LL + lane < n) ? A.row_len[last * 32LL + lane] : 0;
        lastn = __reduce_add_sync(0xFFFFFFFFu, lastn);
        const int64_t ent = vs[last] + lastn;
        if (lane == 0) {
            hd[4 + j] = vo;
            if (j == 0) {
                hd[0] = cs[c];
                hd[1] = ns;
                hd[2] = (int32_t)ent;
            }
        }
        bb[16 + 4 * ns + 32 * j + lane] = (uint8_t)len;
        double *bv = (double *)(bb + sellv_hdr_bytes(ns));
        int32_t *bx = (int32_t *)(bv + ent);
        const int64_t so = A.slice_off[s];
        int off = vo;
        for (int k = 0; k < W; ++k) {
            const unsigned m = __ballot_sync(0xFFFFFFFFu, k < len);
            if (k < len) {
                const int d = off + __popc(m & ((1u << lane) - 1u));
                bv[d] = A.val[so + 32 * k + lane];
                bx[d] = A.col[so + 32 * k + lane];
            }
            off += __popc(m);
        }
    }
}

// x-buffer index range of each slice's nonzeros (lo = INT32_MAX, hi = -1 if none)
__global__ void sellv_xrange_kernel(int64_t n, int64_t nslices, SellMat A, int32_t *lo, int32_t *hi) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t s = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; s < nslices; s += nw) {
        const int64_t pos = s * 32 + lane, so = A.slice_off[s];
        const int len = pos < n ? A.row_len[pos] : 0;
        int mn = INT32_MAX, mx = -1;
        for (int k = 0; k < len; ++k) {
            const int i = (int)(pos + A.col[so + 32 * k + lane]);
            mn = min(mn, i);
            mx = max(mx, i);
        }
        mn = (int)__reduce_min_sync(0xFFFFFFFFu, (unsigned)mn);
        mx = __reduce_max_sync(0xFFFFFFFFu, mx);
        if (lane == 0) {
            lo[s] = mn;
            hi[s] = mx < 0 ? -1 : mx + 1;
        }
    }
}

// The x window.  A CTA folds a contiguous run of chunks (the rows of a banded
// matrix advance with it), so the x entries its chunks read form a sliding
// window: the producer streams x into a ring of XR doubles (XR a power of
// of 64; entry i at slot i mod XR) ahead of each chunk -- [loaded, hi'_c),
// hi'_c = the running maximum of the chunks' upper x indices -- on the same
// mbarrier as the chunk.  Setup checks that no chunk in flight can see its
// entries overwritten (hi'_{c+STAGES-1} - lo_c <= XR - 4) with at least
// PV_MIN_WIN_STAGES ring stages, else this kernel is not used.  The consumers
// gather from shared memory: x crosses HBM/L2 about once instead of once per
// nonzero.  Measured alternatives: the same ring with x
// gathered through L1/L2 runs at 0.45-0.75x the row-per-thread kernel (16
// warps cannot cover the gather latency); with C4's +-5000 band the window
// takes 128 KB and leaves 4 stages: 340 us vs 308 us row-per-thread, so C4
// stays on the row-per-thread kernel; a +-1000 band: 233 us vs 285 us.
template <int MODE, int NCW, int UNR, bool GLD, bool PF = false>
__global__ void __launch_bounds__((NCW + 1) * 32, 1)
    spmv_sellv_kernel(int64_t n, const unsigned char *__restrict__ blob, const int64_t *__restrict__ blob_off,
                      const int32_t *__restrict__ clo, const int32_t *__restrict__ chi,
                      const int32_t *__restrict__ perm, const double *__restrict__ x, double *__restrict__ y,
                      const double *__restrict__ b, double *__restrict__ y2, const Scalars *sc, int STAGE, int STAGES,
                      int XR, int64_t cbeg, int64_t cend) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    double *xw = (double *)(smem_raw + (size_t)STAGES * STAGE);
    uint64_t *full = (uint64_t *)(xw + XR);
    uint64_t *empty = full + STAGES;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const unsigned lt = (1u << lane) - 1u;
    // this CTA's contiguous run of chunks
    const int64_t U = cend - cbeg;
    const int64_t c0 = cbeg + U * blockIdx.x / gridDim.x, c1 = cbeg + U * (blockIdx.x + 1) / gridDim.x;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NCW);
        }
        mbar_fence_init();
    }
    __syncthreads();
    if (warp == NCW) {  // producer warp
        int mn = INT32_MAX;
        for (int64_t c = c0 + lane; c < c1; c += 32) mn = min(mn, __ldg(&clo[c]));
        mn = (int)__reduce_min_sync(0xFFFFFFFFu, (unsigned)mn);
        if (lane == 0) {
            const int start = mn == INT32_MAX ? 0 : (mn & ~1);
            int loaded = start;  // x entries [start, loaded) went out
            // x range of chunk c given what went out before it (even bounds: 16-byte copies)
            auto need = [&](int64_t c, int ld) { return max(ld, (__ldg(&chi[c]) + 1) & ~1); };
            auto xcopy = [&](int a, int e, uint64_t *bar) {  // x[a, e) -> ring, split at the wrap
                while (a < e) {
                    const int sl = a % XR, m = min(e - a, XR - sl);
                    bulk_g2s(xw + sl, x + a, (uint32_t)m * 8u, bar);
                    a += m;
                }
            };
            int st = 0, issued = 0;
            uint32_t ph = 0;
            bool ok = true, gated = false;
            const uint64_t pol = l2_policy_evict_first();
            // the PDL wait, then the x ranges of the `cnt` chunks whose matrix
            // went out before it (their bytes are already expected)
            auto open_gate = [&](int cnt) {
                gated = true;
                pdl_sync();
                ok = !(sc && sc->done);
                int ld = start;
                for (int k = 0; k < cnt; ++k) {
                    const int e = need(c0 + k, ld);
                    xcopy(ld, e, &full[k]);
                    ld = e;
                }
            };
            for (int64_t c = c0; c < c1; ++c) {
                if (!gated && issued == STAGES) {
                    open_gate(STAGES);
                    if (!ok) break;
                }
                // GLD: the chunk's header only (STAGE bytes; the blob has that much slack)
                const int64_t o0 = __ldg(&blob_off[c]), o1 = GLD ? o0 + STAGE : __ldg(&blob_off[c + 1]);
                const int e = need(c, loaded);
                mbar_wait(&empty[st], ph ^ 1u);
                mbar_expect_tx(&full[st], (uint32_t)(o1 - o0) + (uint32_t)(e - loaded) * 8u);
                bulk_g2s_stream(smem_raw + (size_t)st * STAGE, blob + o0, (uint32_t)(o1 - o0), &full[st], pol);
                if (gated) xcopy(loaded, e, &full[st]);
                loaded = e;
                ++issued;
                if (++st == STAGES) {
                    st = 0;
                    ph ^= 1u;
                }
            }
            if (!gated) open_gate(issued);  // run of at most STAGES chunks
            if (!ok)  // aborted (solve already done): drain what went out
                for (int k = 0; k < min(issued, STAGES); ++k) mbar_wait(&full[k], 0u);
        }
        __syncwarp();
        return;
    }
    pdl_sync();
    if (sc && sc->done) return;
    int st = 0, rot = 0;
    uint32_t ph = 0;
    for (int64_t c = c0; c < c1; ++c) {
        mbar_wait(&full[st], ph);
        const unsigned char *sb = smem_raw + (size_t)st * STAGE;
        const int32_t *hd = (const int32_t *)sb;
        const int ns = hd[1];
        int j = warp - rot;
        if (j < 0) j += NCW;
        if (j < ns) {
            const int nval = hd[2];
            const int len = sb[16 + 4 * ns + 32 * j + lane];
            const int W = (int)__reduce_max_sync(0xFFFFFFFFu, (unsigned)len);
            // values and column ids: in the stage, or (GLD) streamed from the blob
            const double *vs = (const double *)((GLD ? blob + __ldg(&blob_off[c]) : sb) + sellv_hdr_bytes(ns));
            const int32_t *xs = (const int32_t *)(vs + nval);
            const int64_t pos = ((int64_t)hd[0] + j) * 32 + lane;
            const int lo = __ldg(&clo[c]);
            const int ipos = (int)pos - (lo - lo % XR);  // slot of x entry i: i - base, minus XR once if past the ring
            int off = hd[4 + j];
            double acc = 0.0;
            // slots k..k+UNR-1: this lane's entry ranks (ballots, no data
            // dependence), their values and column ids, then the x gathers
            // from the window and the ordered fma chain (R-6, +0.0 start)
            auto load = [&](int k, int (&cc)[UNR], double (&vv)[UNR]) {
                int d[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u) {  // slot k+u: this lane's rank among the active lanes
                    const unsigned m = __ballot_sync(0xFFFFFFFFu, k + u < len);
                    d[u] = off + __popc(m & lt);
                    off += __popc(m);
                }
#pragma unroll
                for (int u = 0; u < UNR; ++u)
                    if (k + u < len) {
                        cc[u] = GLD ? __ldcs(xs + d[u]) : xs[d[u]];
                        vv[u] = GLD ? __ldcs(vs + d[u]) : vs[d[u]];
                    }
            };
            auto fold = [&](int k, const int (&cc)[UNR], const double (&vv)[UNR]) {
                double xv[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u)
                    if (k + u < len) {
                        int sl = ipos + cc[u];
                        if (sl >= XR) sl -= XR;
                        xv[u] = xw[sl];
                    }
#pragma unroll
                for (int u = 0; u < UNR; ++u)
                    if (k + u < len) acc = __fma_rn(vv[u], xv[u], acc);
            };
            if constexpr (PF) {  // software pipeline: the next slots' loads are in flight during a fold
                int ca[UNR], cb[UNR];
                double va[UNR], vb[UNR];
                if (W > 0) load(0, ca, va);
                for (int k = 0; k < W; k += 2 * UNR) {
                    if (k + UNR < W) load(k + UNR, cb, vb);
                    fold(k, ca, va);
                    if (k + 2 * UNR < W) load(k + 2 * UNR, ca, va);
                    if (k + UNR < W) fold(k + UNR, cb, vb);
                }
            } else {
                for (int k = 0; k < W; k += UNR) {
                    int cc[UNR];
                    double vv[UNR];
                    load(k, cc, vv);
                    fold(k, cc, vv);
                }
            }
            if (pos < n) {
                const int64_t row = perm ? (int64_t)__ldg(&perm[pos]) : pos;
                if (MODE == SPMV_PLAIN) {
                    y[row] = acc;
                } else {
                    const double r = __dsub_rn(b[row], acc);  // r0 := b - A x0 (l.64)
                    y[row] = r;
                    if (y2) y2[row] = r;
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[st]);
        // a full chunk shifts the assignment by one more warp: slice j of
        // every sigma window (rows sorted by length) visits every warp
        rot += ns == NCW ? ns + 1 : ns;
        if (rot >= NCW) rot -= NCW;
        if (rot >= NCW) rot -= NCW;
        if (++st == STAGES) {
            st = 0;
            ph ^= 1u;
        }
    }
}

}  // namespace pbcg
