// exblas.cuh -- ExBLAS-style exactly rounded dot products on sm_100a.
//
// PAPER.md §2 l.95: "ExBLAS combines together long accumulator and
// floating-point expansions"; results are "independent of data partitioning,
// order of computations, thread scheduling, or reduction tree schemes".
// SPEC.md l.116-117 fixes the two-level scheme (per-element TwoProd, an FPE of
// doubles fed by TwoSum, spill into a Kulisch long accumulator, one rounding).
//
// B200 placement:
//   registers  per thread and per dot, two FPEs: P (the rounded products
//              p = fl(x*y)) and E (their exact errors e = x*y - p), NP/NE
//              doubles each, fed by branch-free Knuth TwoSum;
//   shared     a residual that falls out of an FPE is deposited into the
//              CTA's superaccumulator with int64 shared atomics (rare);
//   warp       at the end the lanes' FPEs are merged into lane 0 by a
//              shuffle tree (TwoSum again; exact), lane 0 deposits its terms;
//   CTA        the CTA normalises its superaccumulator and red.adds the
//              nonzero words into a global one;
//   grid       the last CTA (ticket) normalises and rounds once (or, with
//              several ranks, leaves the normalised words for the int64
//              allreduce).
// Invariant: value(FPEs) + value(superaccumulators) + unread inputs = the
// exact sum, at every point -- so the result is the exact sum rounded once,
// whatever the grid, the thread order, NP/NE or the number of ranks.
//
// Superaccumulator geometry: SACC_L int64 words holding 32-bit digits, bit 0
// of word 0 weighs 2^-1074 (the binary64 LSB), so any double deposits into at
// most 3 words without carries; 31 spare bits per word absorb 2^31 deposits.
// Normalised form: words 0..L-2 in [0,2^32), word L-1 signed.  Range: up to
// 2^(32*66 - 1074 + 63) -- far beyond any sum of < 2^40 products < 2^1000.
#pragma once
#include <cstdint>
#include <cstring>

namespace pbcg {

constexpr int SACC_L = 67;
constexpr int SACC_FLAGW = 2;  // two trailing words: #CTAs with a range flag, with a non-finite flag

enum : unsigned { FLAG_RANGE = 1u, FLAG_NONFINITE = 2u };

// Diagnostic counters (built only with -DPBCG_DEBUG_COUNTERS): spill events
// per kernel family, read back with pbcg_debug_counters().
__device__ unsigned long long g_dbg[16];
#ifdef PBCG_DEBUG_COUNTERS
#define PBCG_COUNT(i) atomicAdd(&g_dbg[(i)], 1ull)
// phase timestamps (globaltimer, ns) of thread 0 of block 0: slots 8..12
#define PBCG_TS(k)                                                                     \
    do {                                                                               \
        if ((threadIdx.x & 31) == 0) {                                                 \
            unsigned long long t_;                                                     \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
            atomicMax(&g_dbg[8 + (k)], t_);                                            \
        }                                                                              \
    } while (0)
#else
#define PBCG_COUNT(i) ((void)0)
#define PBCG_TS(k) ((void)0)
#endif
// Per-CTA timeline (built only with -DPBCG_TIMELINE; tools/timeline.py):
// globaltimer of thread 0 at phase k of kernel kind (0 K2, 1 SpMV, 2 K3)
__device__ unsigned long long g_tl[3][256][8];
#ifdef PBCG_TIMELINE
#define PBCG_TL(kind, k)                                                               \
    do {                                                                               \
        if (threadIdx.x == 0 && blockIdx.x < 256) {                                    \
            unsigned long long t_;                                                     \
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                     \
            g_tl[(kind)][blockIdx.x][(k)] = t_;                                        \
        }                                                                              \
    } while (0)
#else
#define PBCG_TL(kind, k) ((void)0)
#endif

// Programmatic dependent launch: a kernel launched with programmatic stream
// serialisation may start while the previous kernel of the stream finishes;
// griddepcontrol.wait blocks until that kernel has completed and its memory
// is visible, so everything before it (barrier init, smem zeroing, the CTA
// getting resident) overlaps the previous kernel's tail.  launch_dependents
// lets the next such kernel start likewise.  Both are no-ops without PDL.
__device__ __forceinline__ void pdl_sync() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
// wait only: for a kernel of many waves, an early trigger would let the next
// (persistent, shared-memory-heavy) kernel occupy SMs its last waves need
// (measured on C4: 1316 -> 1164 iter/s); dependents start at its exit instead
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void two_sum(double a, double b, double &s, double &e) {
    // Knuth TwoSum, 6 DADD, exact for all finite a, b without overflow.
    s = __dadd_rn(a, b);
    double bp = __dsub_rn(s, a);
    double ap = __dsub_rn(s, bp);
    e = __dadd_rn(__dsub_rn(a, ap), __dsub_rn(b, bp));
}

__device__ __forceinline__ bool is_nonzero(double v) { return (__double_as_longlong(v) << 1) != 0; }
__device__ __forceinline__ bool is_zero(double v) { return (__double_as_longlong(v) << 1) == 0; }
__device__ __forceinline__ bool any_nonzero(const double *v, int n) {
    unsigned long long acc = 0;
#pragma unroll
    for (int i = 0; i < n; ++i) acc |= (unsigned long long)__double_as_longlong(v[i]) << 1;
    return acc != 0;
}

__host__ __device__ __forceinline__ double bits_to_double(unsigned long long b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double((long long)b);
#else
    double d;
    memcpy(&d, &b, 8);
    return d;
#endif
}
__host__ __device__ __forceinline__ int clz32(unsigned v) {
#ifdef __CUDA_ARCH__
    return __clz(v);
#else
    return __builtin_clz(v);
#endif
}

__host__ __device__ __forceinline__ long long double_to_bits(double v) {
#ifdef __CUDA_ARCH__
    return __double_as_longlong(v);
#else
    long long b;
    memcpy(&b, &v, 8);
    return b;
#endif
}

// Split a finite double into signed 32-bit-digit chunks (c0,c1,c2) for words
// i, i+1, i+2 of the superaccumulator.  Returns false for NaN/Inf (which the
// callers flag and never deposit).
__host__ __device__ __forceinline__ bool sacc_split(double v, int &i, long long &c0, long long &c1, long long &c2) {
    const long long bits = double_to_bits(v);
    const unsigned E = (unsigned)(bits >> 52) & 0x7FFu;
    if (E == 0x7FFu) return false;
    unsigned long long m = (unsigned long long)bits & 0xFFFFFFFFFFFFFull;
    int off = 0;
    if (E) { m |= (1ull << 52); off = (int)E - 1; }  // LSB exponent E-1075 -> bit E-1 above 2^-1074
    i = off >> 5;
    const int s = off & 31;
    const unsigned long long sh = m << s;
    c0 = (long long)(sh & 0xFFFFFFFFull);
    c1 = (long long)(sh >> 32);
    c2 = s ? (long long)(m >> (64 - s)) : 0ll;
    if (bits < 0) { c0 = -c0; c1 = -c1; c2 = -c2; }
    return true;
}

// Add a signed 64-bit value c to a 64-bit shared word using native 32-bit
// shared atomics (sm_100 has no 64-bit shared atomic add; atomicAdd(u64*) on
// shared memory compiles to a CAS loop).  The word is (lo, hi) little-endian;
// the carry/borrow out of lo is derived from the value the atomic returned,
// so concurrent additions stay exact (mod 2^64, i.e. two's complement).
__device__ __forceinline__ void sacc_add_shared(unsigned long long *word, long long c) {
    unsigned *p = reinterpret_cast<unsigned *>(word);
    const unsigned lo_add = (unsigned)(unsigned long long)c;
    const unsigned old = atomicAdd(p, lo_add);
    const unsigned carry = ((unsigned long long)old + lo_add) >> 32;  // 0 or 1
    const unsigned hi_add = (unsigned)(c >> 32) + carry;                  // -1, 0 or 1 (mod 2^32)
    if (hi_add) atomicAdd(p + 1, hi_add);
}

// Deposit a finite double into a superaccumulator in shared memory (the
// rare path: kept out of line so the streaming loops stay small).
__device__ __noinline__ void sacc_deposit(unsigned long long *acc, double v) {
    PBCG_COUNT(3);
    int i;
    long long c0, c1, c2;
    if (!sacc_split(v, i, c0, c1, c2)) return;
    if (c0) sacc_add_shared(&acc[i], c0);
    if (c1) sacc_add_shared(&acc[i + 1], c1);
    if (c2) sacc_add_shared(&acc[i + 2], c2);
}

// Host twin (CPU-side tests of the rounding path and of cross-rank merging).
inline void sacc_deposit_host(long long *acc, double v) {
    int i;
    long long c0, c1, c2;
    if (!sacc_split(v, i, c0, c1, c2)) return;
    acc[i] += c0;
    acc[i + 1] += c1;
    acc[i + 2] += c2;
}

// Carry-normalise (one thread): words 0..L-2 -> [0,2^32), carry into word L-1.
__host__ __device__ __forceinline__ void sacc_normalize(long long *w) {
    long long carry = 0;
#pragma unroll 8
    for (int i = 0; i < SACC_L - 1; ++i) {
        long long v = w[i] + carry;
        carry = v >> 32;  // arithmetic shift = floor division
        w[i] = v & 0xFFFFFFFFll;
    }
    w[SACC_L - 1] += carry;
}

// bit `k` of a little-endian array of 32-bit digits
__host__ __device__ __forceinline__ unsigned dig_bit(const unsigned *d, int k) { return (d[k >> 5] >> (k & 31)) & 1u; }

// Round a NORMALISED superaccumulator to the nearest binary64, ties to even.
// Exact zero -> +0.0.  Overflow -> +-inf and *ovf = true.
__host__ __device__ inline double sacc_round(const long long *w, bool *ovf) {
    constexpr int ND = SACC_L + 1;  // digits 0..L-2 from words, L-1 and L from the signed top word
    unsigned d[ND];
    for (int i = 0; i < SACC_L - 1; ++i) d[i] = (unsigned)w[i];
    const long long top = w[SACC_L - 1];
    d[SACC_L - 1] = (unsigned)((unsigned long long)top & 0xFFFFFFFFull);
    d[SACC_L] = (unsigned)((unsigned long long)top >> 32);
    const bool neg = top < 0;
    if (neg) {  // two's complement negation of the ND-digit number
        unsigned long long c = 1;
        for (int i = 0; i < ND; ++i) {
            unsigned long long t = (unsigned long long)(~d[i]) + c;
            d[i] = (unsigned)t;
            c = t >> 32;
        }
    }
    int hi = ND - 1;
    while (hi >= 0 && d[hi] == 0) --hi;
    if (hi < 0) return 0.0;
    const int B = hi * 32 + 31 - clz32(d[hi]);  // index of the most significant bit (bit 0 = 2^-1074)
    double r;
    if (B < 52) {  // subnormal range: every multiple of 2^-1074 below 2^-1022 is exact
        unsigned long long m = 0;
        for (int k = B; k >= 0; --k) m = (m << 1) | dig_bit(d, k);
        r = bits_to_double(m);  // subnormal encoding = integer multiple of 2^-1074
    } else {
        int k0 = B - 52;  // kept LSB
        unsigned long long m = 0;
        for (int k = B; k >= k0; --k) m = (m << 1) | dig_bit(d, k);
        unsigned rb = (k0 >= 1) ? dig_bit(d, k0 - 1) : 0u;
        bool sticky = false;
        if (k0 >= 2) {
            const int lim = k0 - 1;  // bits [0, lim) below the round bit
            for (int i = 0; i < (lim >> 5) && !sticky; ++i) sticky = d[i] != 0;
            if (!sticky && (lim & 31)) sticky = (d[lim >> 5] & ((1u << (lim & 31)) - 1u)) != 0;
        }
        if (rb && (sticky || (m & 1ull))) {
            m += 1;
            if (m == (1ull << 53)) { m >>= 1; k0 += 1; }
        }
        // value = m * 2^(k0 - 1074), m in [2^52, 2^53): biased exponent = k0 + 1
        const long long be = (long long)k0 + 1;
        if (be >= 2047) {
            *ovf = true;
            r = bits_to_double(0x7FF0000000000000ull);
        } else {
            r = bits_to_double(((unsigned long long)be << 52) | (m & 0xFFFFFFFFFFFFFull));
        }
    }
    return neg ? -r : r;
}

// Warp-parallel twin of sacc_round (all 32 lanes; same result in every lane).
// Digits are spread over the lanes (digit i in lane i%32, slot i/32); the
// sign, the lowest / highest nonzero digit and the sticky bit come from
// ballots, so the cost is a few dozen instructions instead of a serial scan.
__device__ double sacc_round_warp(const long long *w, bool *ovf) {
    const int lane = threadIdx.x & 31;
    constexpr int ND = SACC_L + 1;  // 68 two's complement 32-bit digits
    const long long top = w[SACC_L - 1];
    unsigned dg[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const int i = lane + 32 * k;
        dg[k] = i < SACC_L - 1 ? (unsigned)w[i]
                : i == SACC_L - 1 ? (unsigned)((unsigned long long)top & 0xFFFFFFFFull)
                : i == SACC_L ? (unsigned)((unsigned long long)top >> 32) : 0u;
    }
    auto lowest = [&](const unsigned *m) -> int {
        for (int k = 0; k < 3; ++k)
            if (m[k]) return 32 * k + __ffs(m[k]) - 1;
        return -1;
    };
    unsigned msk[3];
    if (top < 0) {  // magnitude = two's complement negation: ~d + 1 rippling from the lowest nonzero digit
#pragma unroll
        for (int k = 0; k < 3; ++k) msk[k] = __ballot_sync(0xFFFFFFFFu, dg[k] != 0u);
        const int z = lowest(msk);
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            const int i = lane + 32 * k;
            dg[k] = i >= ND ? 0u : (i < z) ? 0u : (i == z) ? (0u - dg[k]) : ~dg[k];
        }
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) msk[k] = __ballot_sync(0xFFFFFFFFu, dg[k] != 0u);
    int H = -1;
    for (int k = 2; k >= 0 && H < 0; --k)
        if (msk[k]) H = 32 * k + 31 - __clz(msk[k]);
    if (H < 0) return 0.0;
    auto get = [&](int i) -> unsigned {  // digit i, i uniform across the warp
        const int kk = i < 0 ? 0 : i >> 5;
        const unsigned v = kk == 0 ? dg[0] : kk == 1 ? dg[1] : dg[2];
        const unsigned r = __shfl_sync(0xFFFFFFFFu, v, i < 0 ? 0 : (i & 31));
        return i < 0 ? 0u : r;
    };
    const unsigned hi = get(H), mid = get(H - 1), lo = get(H - 2);
    bool below = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) below |= __any_sync(0xFFFFFFFFu, dg[k] != 0u && (lane + 32 * k) < H - 2);
    const int p = 31 - __clz(hi);
    const int B = 32 * H + p;  // index of the most significant bit (bit 0 = 2^-1074)
    double r;
    if (B < 52) {  // subnormal: exact, digits 0 and 1 only
        const unsigned long long m = ((unsigned long long)get(1) << 32) | get(0);
        r = bits_to_double(m);
    } else {
        const int sft = 31 - p;
        const unsigned long long top64 = ((unsigned long long)hi << 32) | mid;
        const unsigned long long T = sft ? ((top64 << sft) | ((unsigned long long)lo >> (32 - sft))) : top64;
        const unsigned rest = sft ? (unsigned)(lo << sft) : lo;
        unsigned long long m = T >> 11;  // 53 bits, MSB at bit 52
        const unsigned rb = (unsigned)(T >> 10) & 1u;
        const bool sticky = ((T & 0x3FFull) != 0) || rest != 0 || below;
        int k0 = B - 52;
        if (rb && (sticky || (m & 1ull))) {
            m += 1;
            if (m == (1ull << 53)) { m >>= 1; k0 += 1; }
        }
        const long long be = (long long)k0 + 1;
        if (be >= 2047) {
            *ovf = true;
            r = bits_to_double(0x7FF0000000000000ull);
        } else {
            r = bits_to_double(((unsigned long long)be << 52) | (m & 0xFFFFFFFFFFFFFull));
        }
    }
    return top < 0 ? -r : r;
}

template <int N>
struct Fpe {
    double a[N];
    __device__ __forceinline__ void zero() {
#pragma unroll
        for (int i = 0; i < N; ++i) a[i] = 0.0;
    }
    // cascade v through the expansion; returns what did not fit (exactly)
    __device__ __forceinline__ double add(double v) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            double s, e;
            two_sum(a[i], v, s, e);
            a[i] = s;
            v = e;
        }
        return v;
    }
    // same, but stops once the carried value is zero in every lane of the
    // warp (warp-uniform branch; all 32 lanes must be active)
    __device__ __forceinline__ double add_early(double v) {
#pragma unroll
        for (int i = 0; i < N; ++i) {
            if (i >= 2 && !__any_sync(0xFFFFFFFFu, is_nonzero(v))) break;
            double s, e;
            two_sum(a[i], v, s, e);
            a[i] = s;
            v = e;
        }
        return v;
    }
};

// Range rule (R-9): with x,y != 0, flag when |fl(x*y)| < 2^-960 or
// >= 2^1000 (TwoProd is exact outside that zone); NaN/Inf flagged non-finite.
__device__ __noinline__ unsigned range_class(double x, double y) {
    const bool xz = (__double_as_longlong(x) << 1) == 0, yz = (__double_as_longlong(y) << 1) == 0;
    const unsigned ex = (unsigned)(__double_as_longlong(x) >> 52) & 0x7FFu;
    const unsigned ey = (unsigned)(__double_as_longlong(y) >> 52) & 0x7FFu;
    if (ex == 0x7FFu || ey == 0x7FFu) return FLAG_NONFINITE;
    if (xz || yz) return 0u;
    return FLAG_RANGE;
}

template <int NP, int NE>
struct ExAcc {
    Fpe<NP> P;
    Fpe<NE> E;
    __device__ __forceinline__ void zero() {
        P.zero();
        E.zero();
    }
    // acc += x*y exactly; residuals go to the shared superaccumulator `sacc`.
    // EARLY (warp-uniform early exit) requires all 32 lanes to be active.
    template <bool EARLY = true>
    __device__ __forceinline__ void add(double x, double y, unsigned long long *sacc, unsigned &flags) {
        const double p = __dmul_rn(x, y);
        const double e = __fma_rn(x, y, -p);
        const unsigned ep = (unsigned)(__double2hiint(p) >> 20) & 0x7FFu;
        if (ep - 63u >= 1960u) flags |= range_class(x, y);
        double r = EARLY ? P.add_early(p) : P.add(p);
        if (is_nonzero(r)) sacc_deposit(sacc, r);
        r = EARLY ? E.add_early(e) : E.add(e);
        if (is_nonzero(r)) sacc_deposit(sacc, r);
    }
    // merge the lanes of the warp into lane 0 (tree: at step `off` lanes
    // [0,off) absorb lanes [off,2off); the senders' terms are then dead)
    __device__ __forceinline__ void warp_merge(unsigned long long *sacc) {
        const int lane = threadIdx.x & 31;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            double ip[NP], ie[NE];
#pragma unroll
            for (int j = 0; j < NP; ++j) ip[j] = __shfl_down_sync(0xFFFFFFFFu, P.a[j], off);
#pragma unroll
            for (int j = 0; j < NE; ++j) ie[j] = __shfl_down_sync(0xFFFFFFFFu, E.a[j], off);
            if (lane < off) {
#pragma unroll
                for (int j = 0; j < NP; ++j) {
                    double r = P.add(ip[j]);
                    if (is_nonzero(r)) sacc_deposit(sacc, r);
                }
#pragma unroll
                for (int j = 0; j < NE; ++j) {
                    double r = E.add(ie[j]);
                    if (is_nonzero(r)) sacc_deposit(sacc, r);
                }
            }
        }
        if (lane == 0) {
#pragma unroll
            for (int j = 0; j < NP; ++j)
                if (is_nonzero(P.a[j])) sacc_deposit(sacc, P.a[j]);
#pragma unroll
            for (int j = 0; j < NE; ++j)
                if (is_nonzero(E.a[j])) sacc_deposit(sacc, E.a[j]);
        }
    }
};

// Deposit every nonzero residual of a batch (the rare path).
__device__ __forceinline__ void deposit_residuals(const double *res, int n, unsigned long long *sacc) {
#pragma unroll
    for (int i = 0; i < n; ++i)
        if (is_nonzero(res[i])) sacc_deposit(sacc, res[i]);
}

// Exact warp sum of digit chunks with two REDUX.SUM.  Result valid in every lane.
__device__ __forceinline__ long long warp_sum_i64(long long v) {
    // |v| < 2^32 (a digit chunk of sacc_split, possibly negated): a 16-bit
    // unsigned low limb and a signed high limb; 32 lanes sum each limb
    // without overflow (2^21), so two REDUX give the exact sum.
    const unsigned lo = __reduce_add_sync(0xFFFFFFFFu, (unsigned)((unsigned long long)v & 0xFFFFu));
    const int hi = __reduce_add_sync(0xFFFFFFFFu, (int)(v >> 16));
    return (long long)hi * 65536 + (long long)lo;
}

// Deposit one double per lane (zeros allowed) into a shared superaccumulator.
// When the warp's values touch at most 4 consecutive words (the usual case:
// the lanes' expansion terms have similar exponents), the chunks are summed
// across the warp first and lane 0 adds 4 words -- no same-address atomic
// storms; otherwise every lane deposits its own value.  All 32 lanes active.
__device__ __forceinline__ void warp_deposit(double v, unsigned long long *sacc) {
    int i = 0;
    long long c0 = 0, c1 = 0, c2 = 0;
    const bool nz = is_nonzero(v) && sacc_split(v, i, c0, c1, c2);
    const unsigned imin = __reduce_min_sync(0xFFFFFFFFu, nz ? (unsigned)i : 0xFFFFFFFFu);
    if (imin == 0xFFFFFFFFu) return;  // all lanes zero
    const unsigned imax = __reduce_max_sync(0xFFFFFFFFu, nz ? (unsigned)i : 0u);
    if (imax - imin <= 1u && imin + 3u < (unsigned)SACC_L) {
        const bool sh = nz && ((unsigned)i != imin);
        if (!nz) { c0 = 0; c1 = 0; c2 = 0; }
        const long long d0 = sh ? 0 : c0, d1 = sh ? c0 : c1, d2 = sh ? c1 : c2, d3 = sh ? c2 : 0;
        const long long s0 = warp_sum_i64(d0), s1 = warp_sum_i64(d1), s2 = warp_sum_i64(d2), s3 = warp_sum_i64(d3);
        if ((threadIdx.x & 31) == 0) {
            if (s0) sacc_add_shared(&sacc[imin], s0);
            if (s1) sacc_add_shared(&sacc[imin + 1], s1);
            if (s2) sacc_add_shared(&sacc[imin + 2], s2);
            if (s3) sacc_add_shared(&sacc[imin + 3], s3);
        }
    } else if (nz) {
        sacc_deposit(sacc, v);
    }
}

// The same into words private to this warp (`w`, int64, e.g. a drained ring
// area): lane 0 adds the warp sums with plain 64-bit adds -- no atomics, and
// no contention with the other warps of the CTA (their deposits of similar
// exponents would hit the same few words); the rare wide case deposits per
// lane with the 32-bit atomics, which only this warp's lanes race on.
__device__ __forceinline__ void warp_deposit_priv(double v, long long *w) {
    int i = 0;
    long long c0 = 0, c1 = 0, c2 = 0;
    const bool nz = is_nonzero(v) && sacc_split(v, i, c0, c1, c2);
    const unsigned imin = __reduce_min_sync(0xFFFFFFFFu, nz ? (unsigned)i : 0xFFFFFFFFu);
    if (imin == 0xFFFFFFFFu) return;
    const unsigned imax = __reduce_max_sync(0xFFFFFFFFu, nz ? (unsigned)i : 0u);
    if (imax - imin <= 1u && imin + 3u < (unsigned)SACC_L) {
        const bool sh = nz && ((unsigned)i != imin);
        if (!nz) { c0 = 0; c1 = 0; c2 = 0; }
        const long long d0 = sh ? 0 : c0, d1 = sh ? c0 : c1, d2 = sh ? c1 : c2, d3 = sh ? c2 : 0;
        const long long s0 = warp_sum_i64(d0), s1 = warp_sum_i64(d1), s2 = warp_sum_i64(d2), s3 = warp_sum_i64(d3);
        if ((threadIdx.x & 31) == 0) {
            w[imin] += s0;
            w[imin + 1] += s1;
            w[imin + 2] += s2;
            w[imin + 3] += s3;
        }
    } else if (nz) {
        sacc_deposit((unsigned long long *)w, v);
    }
    __syncwarp();
}

// All NT expansion terms of every lane at once (zeros allowed), into words
// private to this warp: when the nonzero terms of the warp span at most
// WIN_W superaccumulator words, every lane adds the digit chunks of its terms
// into ITS OWN column of a WIN_W x 32 window (`win`: WIN_WORDS int64 of
// warp-private shared memory; plain read-modify-writes, no atomics, no
// conflicts between lanes), and lane j then sums row j over the 32 columns
// and adds it to word lo + j -- 2 REDUX for the whole accumulator instead of
// 10 per term (warp_deposit_priv), which the drain was bound by.  Wider
// spreads fall back to one warp_deposit_priv per term.  All 32 lanes active.
#ifndef PBCG_WIN_W
#define PBCG_WIN_W 16
#endif
constexpr int WIN_W = PBCG_WIN_W;         // window rows (superaccumulator words), at most 16
constexpr int WIN_LD = 33;                // row stride in int64: 32 columns + 1 (bank skew for the row sums)
constexpr int WIN_WORDS = WIN_W * WIN_LD;
template <int NT>
__device__ __forceinline__ void warp_window_deposit(const double (&v)[NT], long long *w, long long *win) {
    const int lane = threadIdx.x & 31;
    unsigned lo = 0xFFFFFFFFu, hi = 0u;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        const unsigned E = (unsigned)(__double_as_longlong(v[t]) >> 52) & 0x7FFu;
        if (is_nonzero(v[t]) && E != 0x7FFu) {  // NaN/Inf terms are flagged elsewhere and never deposited (sacc_split)
            const unsigned i = (E ? E - 1u : 0u) >> 5;
            lo = min(lo, i);
            hi = max(hi, i);
        }
    }
    lo = __reduce_min_sync(0xFFFFFFFFu, lo);
    if (lo == 0xFFFFFFFFu) return;  // every term of every lane is zero
    hi = __reduce_max_sync(0xFFFFFFFFu, hi);
    if (hi + 3u - lo > (unsigned)WIN_W) {  // a term touches words i, i+1, i+2
#pragma unroll
        for (int t = 0; t < NT; ++t) warp_deposit_priv(v[t], w);
        return;
    }
    const int span = (int)(hi + 3u - lo);  // window rows in use (warp-uniform)
    long long *col = win + lane;
#pragma unroll
    for (int k = 0; k < WIN_W; ++k)
        if (k < span) col[k * WIN_LD] = 0;
#pragma unroll
    for (int t = 0; t < NT; ++t) {
        int i;
        long long c0, c1, c2;
        if (is_nonzero(v[t]) && sacc_split(v[t], i, c0, c1, c2)) {
            long long *q = col + (i - (int)lo) * WIN_LD;
            q[0] += c0;
            q[WIN_LD] += c1;
            q[2 * WIN_LD] += c2;
        }
    }
    __syncwarp();
    static_assert(WIN_W <= 16, "two lanes per window row");
    const int r = lane & 15;  // lanes r and r + 16 sum the two halves of row r
    long long sum = 0;
    if (r < span) {
        const long long *row = win + r * WIN_LD + (lane & 16);
#pragma unroll
        for (int k = 0; k < 16; ++k) sum += row[k];
    }
    sum += __shfl_xor_sync(0xFFFFFFFFu, sum, 16);
    if (lane < span && lo + (unsigned)lane < (unsigned)SACC_L && sum) w[lo + lane] += sum;
    __syncwarp();
}

// Two-tier accumulator used by the streaming kernels.  Each product p and its
// TwoProd error e enter short hot expansions P, E (NH levels each, branch
// free).  What falls out of them -- values far below this thread's running
// sums, e.g. the 1e-16 interior residue of b = A*ones next to O(1) boundary
// entries, whose products spread over 150-200 bits -- continues into the
// cold levels CP, CE (NC levels each; independent chains for p and e).  One
// warp vote per batch of products decides whether the cold levels run, and a
// second one whether anything fell out of them into the shared
// superaccumulator.  Together the tiers are one exact cascade of NH+NC
// levels per stream; all steps are TwoSums, so tiering only affects speed.
struct Prod {
    double p, e;
};

template <int NH, int NC, int NHE = NH>
struct ExAccT {
    Fpe<NH> P;   // hot levels of the p stream
    Fpe<NHE> E;  // hot levels of the e stream (e sits 53 bits below p: usually needs fewer)
    Fpe<NC> CP, CE;
    __device__ __forceinline__ void zero() {
        P.zero(); E.zero(); CP.zero(); CE.zero();
    }
    // TwoProd + the R-9 range flag (branch free).  zero_op: x or y is +-0.
    __device__ __forceinline__ Prod prep(double x, double y, bool zero_op, unsigned &flags) const {
        Prod r;
        r.p = __dmul_rn(x, y);
        r.e = __fma_rn(x, y, -r.p);
        const unsigned ep = (unsigned)(__double2hiint(r.p) >> 20) & 0x7FFu;
        flags |= (((ep - 63u) >= 1960u) & !zero_op) | (ep == 0x7FFu);
        return r;
    }
    __device__ __forceinline__ void hot(const Prod &q, double *res) {
        res[0] = P.add(q.p);
        res[1] = E.add(q.e);
    }
    __device__ __forceinline__ void cold(const double *in, double *res) {
        res[0] = CP.add(in[0]);
        res[1] = CE.add(in[1]);
    }
    // End of kernel: deposit every expansion term of every lane with one
    // warp-aggregated deposit per term slot (see warp_deposit).
    template <int N>
    __device__ __forceinline__ static void drain_fpe(const Fpe<N> &F, unsigned long long *sacc) {
#pragma unroll
        for (int j = 0; j < N; ++j) warp_deposit(F.a[j], sacc);
    }
    // all 32 lanes of the warp, converged (callers __syncwarp() first)
    __device__ __forceinline__ void warp_merge(unsigned long long *sacc) {
        drain_fpe<NH>(P, sacc);
        drain_fpe<NHE>(E, sacc);
        drain_fpe<NC>(CP, sacc);
        drain_fpe<NC>(CE, sacc);
    }
    // the same into this warp's private words (warp_deposit_priv).  Measured
    // and rejected: cascading the lane's terms into a fresh 3-term expansion
    // first (3 deposits instead of NH + NHE + 2 NC: C3 7,238 vs 7,583 iter/s,
    // one long dependent chain), and batching 2-4 deposits so their REDUX
    // chains interleave (C3 7,218-7,381 vs 7,585).
    // the same through the per-warp window (warp_window_deposit)
    __device__ __forceinline__ void warp_merge_win(long long *w, long long *win) {
        double v[NH + NHE + 2 * NC];
#pragma unroll
        for (int j = 0; j < NH; ++j) v[j] = P.a[j];
#pragma unroll
        for (int j = 0; j < NHE; ++j) v[NH + j] = E.a[j];
#pragma unroll
        for (int j = 0; j < NC; ++j) v[NH + NHE + j] = CP.a[j];
#pragma unroll
        for (int j = 0; j < NC; ++j) v[NH + NHE + NC + j] = CE.a[j];
        warp_window_deposit(v, w, win);
    }
    __device__ __forceinline__ void warp_merge_priv(long long *w) {
#pragma unroll
        for (int j = 0; j < NH; ++j) warp_deposit_priv(P.a[j], w);
#pragma unroll
        for (int j = 0; j < NHE; ++j) warp_deposit_priv(E.a[j], w);
#pragma unroll
        for (int j = 0; j < NC; ++j) warp_deposit_priv(CP.a[j], w);
#pragma unroll
        for (int j = 0; j < NC; ++j) warp_deposit_priv(CE.a[j], w);
    }
};


// Accumulate a batch of K prepared products with one vote per tier.  Product
// k goes to d1 when ALT and k is odd, else to d0 (s0/s1: their shared
// superaccumulators).  All 32 lanes must be active.
template <int K, bool ALT, bool SPLIT = false, class A>
__device__ __forceinline__ void cascade_batch(A &d0, A &d1, const Prod (&P)[K], unsigned long long *s0,
                                              unsigned long long *s1) {
    double rp[K], re[K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double r[2];
        if (ALT && (k & 1)) d1.hot(P[k], r); else d0.hot(P[k], r);
        rp[k] = r[0];
        re[k] = r[1];
    }
    // the p and e streams spill independently (e usually more often: it sits
    // 53 bits below p), so each gets its own vote for its cold levels
    if constexpr (ALT && SPLIT) {  // one vote per (dot, stream): a dot whose residuals are all zero skips its cold levels
        bool any[4] = {false, false, false, false};  // p0, p1, e0, e1
#pragma unroll
        for (int k = 0; k < K; ++k) {
            any[k & 1] |= is_nonzero(rp[k]);
            any[2 + (k & 1)] |= is_nonzero(re[k]);
        }
        const unsigned vp0 = __any_sync(0xFFFFFFFFu, any[0]), vp1 = __any_sync(0xFFFFFFFFu, any[1]);
        const unsigned ve0 = __any_sync(0xFFFFFFFFu, any[2]), ve1 = __any_sync(0xFFFFFFFFu, any[3]);
        if (vp0 | vp1 | ve0 | ve1) {
            PBCG_COUNT(1);
            double cp[K], ce[K];
#pragma unroll
            for (int k = 0; k < K; ++k) {
                cp[k] = 0.0;
                ce[k] = 0.0;
            }
            if (vp0) {
#pragma unroll
                for (int k = 0; k < K; k += 2) cp[k] = d0.CP.add(rp[k]);
            }
            if (vp1) {
#pragma unroll
                for (int k = 1; k < K; k += 2) cp[k] = d1.CP.add(rp[k]);
            }
            if (ve0) {
#pragma unroll
                for (int k = 0; k < K; k += 2) ce[k] = d0.CE.add(re[k]);
            }
            if (ve1) {
#pragma unroll
                for (int k = 1; k < K; k += 2) ce[k] = d1.CE.add(re[k]);
            }
            if (__any_sync(0xFFFFFFFFu, any_nonzero(cp, K) | any_nonzero(ce, K))) {
#pragma unroll
                for (int k = 0; k < K; ++k) {
                    unsigned long long *sk = (k & 1) ? s1 : s0;
                    if (is_nonzero(cp[k])) sacc_deposit(sk, cp[k]);
                    if (is_nonzero(ce[k])) sacc_deposit(sk, ce[k]);
                }
            }
        }
        return;
    }
    const bool cold_p = __any_sync(0xFFFFFFFFu, any_nonzero(rp, K));
    const bool cold_e = __any_sync(0xFFFFFFFFu, any_nonzero(re, K));
    if (cold_p | cold_e) {
        PBCG_COUNT(1);
        double cp[K], ce[K];
#pragma unroll
        for (int k = 0; k < K; ++k) {
            cp[k] = 0.0;
            ce[k] = 0.0;
        }
        if (cold_p) {
#pragma unroll
            for (int k = 0; k < K; ++k) cp[k] = (ALT && (k & 1)) ? d1.CP.add(rp[k]) : d0.CP.add(rp[k]);
        }
        if (cold_e) {
#pragma unroll
            for (int k = 0; k < K; ++k) ce[k] = (ALT && (k & 1)) ? d1.CE.add(re[k]) : d0.CE.add(re[k]);
        }
        if (__any_sync(0xFFFFFFFFu, any_nonzero(cp, K) | any_nonzero(ce, K))) {
#pragma unroll
            for (int k = 0; k < K; ++k) {
                unsigned long long *sk = (ALT && (k & 1)) ? s1 : s0;
                if (is_nonzero(cp[k])) sacc_deposit(sk, cp[k]);
                if (is_nonzero(ce[k])) sacc_deposit(sk, ce[k]);
            }
        }
    }
}

// Same, for lanes that may be inactive or diverged (tails): no votes.
template <class A>
__device__ __forceinline__ void cascade_one(A &d, const Prod &q, unsigned long long *s) {
    double r[2], c[2];
    d.hot(q, r);
    if (any_nonzero(r, 2)) {
        d.cold(r, c);
        deposit_residuals(c, 2, s);
    }
}

// ---------------------------------------------------------------------------
// Plain fp64 accumulation (dot_mode = PBCG_DOT_PLAIN: the
// paper's non-reproducible comparison arm).  Same interface as ExAccT: each
// thread keeps one fma chain per dot, warps reduce by a fixed shuffle tree,
// the CTA sums its warps in order (plain_publish) and the CTA partials are
// summed in grid order by plain_finalize_kernel -- deterministic for one
// launch geometry, but the grouping (hence the bits) follows the partition.
// ---------------------------------------------------------------------------
struct PlainAcc {
    double s;
    int slot;  // this warp's slot in the CTA's per-dot warp sums (-1: unused accumulator)
    __device__ __forceinline__ void zero() { s = 0.0; }
    __device__ __forceinline__ Prod prep(double x, double y, bool, unsigned &) const { return Prod{x, y}; }
    __device__ __forceinline__ void add(const Prod &q) { s = __fma_rn(q.p, q.e, s); }
    __device__ __forceinline__ void warp_merge_priv(long long *) {}
    __device__ __forceinline__ void warp_merge_win(long long *, long long *) {}
    // all 32 lanes, converged: lane 0 stores the warp's sum as a double
    __device__ __forceinline__ void warp_merge(unsigned long long *slots) {
        double v = s;
#pragma unroll
        for (int o = 16; o; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
        if ((threadIdx.x & 31) == 0 && slot >= 0) ((double *)slots)[slot] = v;
    }
};

template <int K, bool ALT, bool SPLIT = false>
__device__ __forceinline__ void cascade_batch(PlainAcc &d0, PlainAcc &d1, const Prod (&P)[K], unsigned long long *,
                                              unsigned long long *) {
#pragma unroll
    for (int k = 0; k < K; ++k) {
        if (ALT && (k & 1)) d1.add(P[k]);
        else d0.add(P[k]);
    }
}

__device__ __forceinline__ void cascade_one(PlainAcc &d, const Prod &q, unsigned long long *) { d.add(q); }

// Shared-memory state of a CTA computing ND dots.
template <int ND>
struct CtaSacc {
    unsigned long long w[ND][SACC_L];
    unsigned flags;
    int last;
    double rounded[ND];
};

template <int ND>
__device__ __forceinline__ void cta_sacc_zero(CtaSacc<ND> &S) {
    for (int i = threadIdx.x; i < ND * SACC_L; i += blockDim.x) (&S.w[0][0])[i] = 0ull;
    if (threadIdx.x == 0) S.flags = 0u;
}

// After every thread has merged its FPEs: normalise the CTA superaccumulators,
// red.add them into gacc[ND*L + FLAGW], take a ticket; returns true in the
// last CTA of the grid (whose threads then see the complete gacc).
template <int ND>
__device__ bool cta_sacc_publish(CtaSacc<ND> &S, unsigned flags, long long *gacc, unsigned *ticket) {
    if (flags) atomicOr(&S.flags, flags);
    __syncthreads();
    if (threadIdx.x < ND) sacc_normalize((long long *)S.w[threadIdx.x]);
    __syncthreads();
    for (int i = threadIdx.x; i < ND * SACC_L; i += blockDim.x) {
        const long long v = (long long)(&S.w[0][0])[i];
        if (v) atomicAdd((unsigned long long *)&gacc[i], (unsigned long long)v);
    }
    if (threadIdx.x == 0) {
        if (S.flags & FLAG_RANGE) atomicAdd((unsigned long long *)&gacc[ND * SACC_L], 1ull);
        if (S.flags & FLAG_NONFINITE) atomicAdd((unsigned long long *)&gacc[ND * SACC_L + 1], 1ull);
    }
    if (!ticket) return false;  // reduced later by finalize_kernel (stream order makes the reds visible)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) S.last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
    __syncthreads();
    if (S.last) __threadfence();
    return S.last != 0;
}

// Plain mode: sum the W warp sums of each dot in order, store the CTA's
// partials part[blockIdx.x * ND + k].
template <int ND, int W>
__device__ void plain_publish(CtaSacc<ND> &S, double *part) {
    __syncthreads();
    if (threadIdx.x < ND) {
        const double *ws = (const double *)S.w[threadIdx.x];
        double t = 0.0;
        for (int i = 0; i < W; ++i) t = __dadd_rn(t, ws[i]);
        part[(size_t)blockIdx.x * ND + threadIdx.x] = t;
    }
}

// In the last CTA: pull gacc into shared memory and normalise it.
template <int ND>
__device__ void cta_sacc_collect(CtaSacc<ND> &S, long long *gacc, unsigned &gflags) {
    long long *w = (long long *)&S.w[0][0];
    for (int i = threadIdx.x; i < ND * SACC_L; i += blockDim.x) w[i] = __ldcg(&gacc[i]);
    __syncthreads();
    if (threadIdx.x < ND) sacc_normalize(w + threadIdx.x * SACC_L);
    __syncthreads();
    const long long fr = __ldcg(&gacc[ND * SACC_L]), fn = __ldcg(&gacc[ND * SACC_L + 1]);
    gflags = (fr ? FLAG_RANGE : 0u) | (fn ? FLAG_NONFINITE : 0u);
}

}  // namespace pbcg
