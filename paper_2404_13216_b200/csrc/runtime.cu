// runtime.cu -- host runtime and C ABI (include/pbicgstab.h) of the B200
// p-BiCGStab + ExBLAS hot path.
//
// Layers:
//   setup    partition / halo plan / sliced-ELL conversion / workspace carve /
//            NCCL communicators (dlopen'ed libnccl.so.2, the copy torch loads)
//   solve    I1-I4 once, then the Algorithm 2 loop replayed as CUDA-graph
//            chunks of `poll_every` iterations; the host polls a device done
//            flag between chunks, later iterations are device-side no-ops
//   ranks    1 rank: K2 -> SpMV(z) -> K3 -> SpMV(w), each dot kernel rounds
//            in its last CTA (no extra launch);
//            P real ranks: phase-A/B superaccumulators allreduced (int64 sum)
//            by NCCL on a side stream while the halo exchange + SpMV run on
//            the main stream (§2 l.90, "communication hiding");
//            V virtual ranks: the same dataflow emulated in one process on
//            one GPU with device copies (partition-invariance test vehicle).
#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <memory>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nccl.h>
#include <nvtx3/nvToolsExt.h>

#include "../../include/pbicgstab.h"
#include "kernels.cuh"
#include "small.cuh"
#include "cluster.cuh"
#include "stream.cuh"

using namespace pbcg;

// ----------------------------------------------------------------------------
// errors
// ----------------------------------------------------------------------------
static thread_local std::string g_err;

static int fail(int rc, const char *fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return rc;
}

#define CUDA_TRY(x)                                                                                      \
    do {                                                                                                 \
        cudaError_t e_ = (x);                                                                            \
        if (e_ != cudaSuccess)                                                                           \
            return fail(PBCG_ECUDA, "%s: %s (%s:%d)", #x, cudaGetErrorString(e_), __FILE__, __LINE__);    \
    } while (0)

#define RC_TRY(x)                  \
    do {                           \
        int rc_ = (x);             \
        if (rc_ != PBCG_OK) return rc_; \
    } while (0)

// NVTX ranges around the host entry points (setup, start, iterate, finish,
// exdot, allreduce enqueue): one nsys capture of a multi-rank run shows the
// reductions beside the SpMV (header-only NVTX 3; no cost without a tool)
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// ----------------------------------------------------------------------------
// NCCL (resolved at run time: the library works without NCCL on one GPU)
// ----------------------------------------------------------------------------
struct NcclApi {
    bool ok = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommInitRankConfig)(ncclComm_t *, int, ncclUniqueId, int, ncclConfig_t *) = nullptr;  // optional
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t *, ncclConfig_t *) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi g_nccl;
static std::once_flag g_nccl_once;

static void nccl_load() {
    const char *names[] = {getenv("PBCG_NCCL_LIB"), "libnccl.so.2", "libnccl.so"};
    void *h = nullptr;
    for (const char *nm : names) {
        if (!nm) continue;
        h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);
        if (!h) h = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (h) break;
    }
    if (!h) return;
#define SYM(f, s) g_nccl.f = (decltype(g_nccl.f))dlsym(h, s)
    SYM(GetUniqueId, "ncclGetUniqueId");
    SYM(CommInitRank, "ncclCommInitRank");
    SYM(CommInitRankConfig, "ncclCommInitRankConfig");
    SYM(CommDestroy, "ncclCommDestroy");
    SYM(CommSplit, "ncclCommSplit");
    SYM(AllReduce, "ncclAllReduce");
    SYM(AllGather, "ncclAllGather");
    SYM(Send, "ncclSend");
    SYM(Recv, "ncclRecv");
    SYM(GroupStart, "ncclGroupStart");
    SYM(GroupEnd, "ncclGroupEnd");
    SYM(GetErrorString, "ncclGetErrorString");
#undef SYM
    g_nccl.ok = g_nccl.GetUniqueId && g_nccl.CommInitRank && g_nccl.CommDestroy && g_nccl.CommSplit && g_nccl.AllReduce &&
                g_nccl.AllGather && g_nccl.Send && g_nccl.Recv && g_nccl.GroupStart && g_nccl.GroupEnd;
}

static bool nccl_available() {
    std::call_once(g_nccl_once, nccl_load);
    return g_nccl.ok;
}

// CTAs per NCCL communicator (ncclConfig_t.maxCTAs): the halo and the
// reduction communicators together fit the SMs the interior SpMV leaves free
static int nccl_ctas() {
    const char *e = getenv("PBCG_NCCL_CTAS");
    return e ? std::max(1, atoi(e)) : 2;
}

#define NCCL_TRY(x)                                                                                          \
    do {                                                                                                     \
        ncclResult_t e_ = (x);                                                                               \
        if (e_ != ncclSuccess)                                                                               \
            return fail(PBCG_ENCCL, "%s: %s", #x, g_nccl.GetErrorString ? g_nccl.GetErrorString(e_) : "?"); \
    } while (0)

// ----------------------------------------------------------------------------
// collective contract of setup: every rank hashes the setup
// arguments that must agree; setup allgathers (row_begin, row_end, hull,
// hash) and every rank checks the same records, so all return the same code
// ----------------------------------------------------------------------------
extern "C" int pbcg_history_digest(const double *hist, int32_t rows, uint64_t *out) {
    if (!out || rows < 0 || (rows > 0 && !hist)) return fail(PBCG_EINVAL, "history_digest: bad arguments");
    constexpr uint64_t B = 0xcbf29ce484222325ull, P = 0x100000001b3ull;  // FNV-1a 64
    uint64_t h = B;
    for (int32_t r = 0; r < rows; ++r) {
        uint64_t rh = B;
        for (int c = 0; c < H_COLS; ++c) {
            uint64_t w;
            memcpy(&w, hist + (size_t)r * H_COLS + c, 8);
            rh = (rh ^ w) * P;
        }
        h = (h ^ rh) * P;
    }
    *out = h;
    return PBCG_OK;
}

extern "C" int pbcg_config_hash(const pbcg_csr_local *A, const pbcg_dist *d, uint64_t *out) {
    if (!out) return fail(PBCG_EINVAL, "config_hash: out == NULL");
    uint64_t hsh = 1469598103934665603ull;  // FNV-1a 64
    auto mix = [&](int64_t v) {
        for (int k = 0; k < 8; ++k) {
            hsh ^= (uint64_t)((v >> (8 * k)) & 0xFF);
            hsh *= 1099511628211ull;
        }
    };
    mix(PBCG_ABI_VERSION);
    mix(A ? A->n_global : -1);  // comm-only handles: no matrix
    mix(d ? std::max(1, d->nranks) : 1);
    mix(d ? std::max(1, d->virtual_ranks) : 1);
    mix(d ? d->precond : 0);
    mix(d ? d->comm_mode : 0);
    *out = hsh;
    return PBCG_OK;
}

// rec: nranks records of PBCG_RANK_REC int64 (row_begin, row_end, cmin, cmax,
// hash); with a matrix the row blocks must tile [0, n_global) in rank order
extern "C" int pbcg_check_ranks(int32_t nranks, const int64_t *rec, int64_t n_global, int32_t has_matrix) {
    if (nranks < 1 || !rec) return fail(PBCG_EINVAL, "check_ranks: bad arguments");
    for (int k = 1; k < nranks; ++k)
        if (rec[PBCG_RANK_REC * k + 4] != rec[4])
            return fail(PBCG_EINVAL, "setup arguments differ between rank 0 and rank %d (config hash)", k);
    if (!has_matrix) return PBCG_OK;
    if (rec[0] != 0) return fail(PBCG_EINVAL, "rank 0 does not start at row 0");
    for (int k = 0; k + 1 < nranks; ++k)
        if (rec[PBCG_RANK_REC * k + 1] != rec[PBCG_RANK_REC * (k + 1)])
            return fail(PBCG_EINVAL, "row blocks of ranks %d and %d are not contiguous", k, k + 1);
    if (rec[PBCG_RANK_REC * (nranks - 1) + 1] != n_global)
        return fail(PBCG_EINVAL, "row blocks of the ranks do not cover [0, n_global)");
    return PBCG_OK;
}

// ----------------------------------------------------------------------------
// host-only planning (exported; CPU-testable)
// ----------------------------------------------------------------------------
extern "C" int pbcg_plan_partition(int64_t n, int32_t p, int64_t *begins) {
    if (n < 0 || p < 1 || !begins) return fail(PBCG_EINVAL, "plan_partition: bad arguments");
    const int64_t q = n / p, rem = n % p;
    begins[0] = 0;
    for (int32_t k = 0; k < p; ++k) begins[k + 1] = begins[k] + q + (k < rem ? 1 : 0);
    return PBCG_OK;
}

static void buf_range(const int64_t *rg, int64_t &lo, int64_t &hi) {
    const int64_t rb = rg[0], re = rg[1], cmin = rg[2], cmax = rg[3];
    lo = rb;
    hi = re;
    if (cmax >= cmin) {
        lo = std::min(lo, cmin);
        hi = std::max(hi, cmax + 1);
    }
}

extern "C" int pbcg_plan_halo(int32_t p, int32_t me, const int64_t *ranges, int64_t *recv_lo, int64_t *recv_hi,
                              int64_t *send_lo, int64_t *send_hi, int64_t *buf_lo, int64_t *buf_hi) {
    if (p < 1 || me < 0 || me >= p || !ranges) return fail(PBCG_EINVAL, "plan_halo: bad arguments");
    for (int32_t q = 0; q < p; ++q) {
        if (ranges[4 * q] > ranges[4 * q + 1]) return fail(PBCG_EINVAL, "plan_halo: rank %d has row_begin > row_end", q);
        if (q > 0 && ranges[4 * q] != ranges[4 * (q - 1) + 1])
            return fail(PBCG_EINVAL, "plan_halo: row blocks do not tile in rank order at rank %d", q);
    }
    int64_t mlo, mhi;
    buf_range(ranges + 4 * me, mlo, mhi);
    if (buf_lo) *buf_lo = mlo;
    if (buf_hi) *buf_hi = mhi;
    const int64_t mrb = ranges[4 * me], mre = ranges[4 * me + 1];
    for (int32_t q = 0; q < p; ++q) {
        int64_t rl = 0, rh = 0, sl = 0, sh = 0;
        if (q != me) {
            const int64_t qrb = ranges[4 * q], qre = ranges[4 * q + 1];
            rl = std::max(mlo, qrb);
            rh = std::min(mhi, qre);
            if (rh <= rl) rl = rh = 0;
            int64_t qlo, qhi;
            buf_range(ranges + 4 * q, qlo, qhi);
            sl = std::max(qlo, mrb);
            sh = std::min(qhi, mre);
            if (sh <= sl) sl = sh = 0;
        }
        if (recv_lo) recv_lo[q] = rl;
        if (recv_hi) recv_hi[q] = rh;
        if (send_lo) send_lo[q] = sl;
        if (send_hi) send_hi[q] = sh;
    }
    return PBCG_OK;
}

// host twins of the device superaccumulator (CPU tests of the merge + round
// path used after the cross-rank allreduce)
extern "C" int pbcg_sacc_accumulate(int64_t n, const double *x, const double *y, int64_t *words) {
    if (n < 0 || !words) return fail(PBCG_EINVAL, "sacc_accumulate: bad arguments");
    long long *w = (long long *)words;
    for (int64_t k = 0; k < n; ++k) {
        const double p = x[k] * y[k];
        const double e = std::fma(x[k], y[k], -p);  // exact in the R-9 zone
        sacc_deposit_host(w, p);
        sacc_deposit_host(w, e);
    }
    sacc_normalize(w);
    return PBCG_OK;
}

extern "C" int pbcg_sacc_round(const int64_t *words, double *out) {
    if (!words || !out) return fail(PBCG_EINVAL, "sacc_round: bad arguments");
    long long w[SACC_L];
    memcpy(w, words, sizeof(w));
    sacc_normalize(w);
    bool ovf = false;
    *out = sacc_round(w, &ovf);
    return ovf ? PBCG_ERANGE : PBCG_OK;
}

extern "C" int pbcg_sacc_words(void) { return SACC_L; }

// ----------------------------------------------------------------------------
// handle
// ----------------------------------------------------------------------------
static constexpr int GW4 = xs_words(4);  // words of a 4-dot reduction buffer (fast words, flags, extended words)
static_assert(GW4 >= XS_GW, "a phase buffer also holds the full-range EXDOT accumulator");
static constexpr int NPH = 5;                        // reduction buffers: init, A, B, true, exdot
static constexpr int K_BS = 256;
static constexpr int PLAIN_GRID = 1024;  // >= any K2/K3 stream grid (one CTA per SM)
static constexpr int K_NP = 4, K_NE = 4;             // FPE depth for products / errors (performance only, R-16)
static constexpr int U_MD4 = 2, U_MD1 = 4;  // row pairs in flight per thread (multidot)

// packed SELL-P geometry (spmv_sellp_kernel): slices per chunk, slices per
// consumer warp, ring stages
#ifndef PBCG_PS_SPS
#define PBCG_PS_SPS 30
#endif
#ifndef PBCG_PS_RPW
#define PBCG_PS_RPW 1
#endif
#ifndef PBCG_PS_MAXSTAGES
#define PBCG_PS_MAXSTAGES 8
#endif
static constexpr int PS_SPS = PBCG_PS_SPS, PS_RPW = PBCG_PS_RPW, PS_MAXSTAGES = PBCG_PS_MAXSTAGES;
static constexpr int PS_SMEM_MAX = 227 * 1024;
// SELL-V geometry (spmv_sellv_kernel, long rows): consumer warps (= most
// slices per chunk), bytes per chunk, gathers in flight per lane, ring stages
#ifndef PBCG_PV_NCW
#define PBCG_PV_NCW 16
#endif
#ifndef PBCG_PV_CAP
#define PBCG_PV_CAP 24576
#endif
#ifndef PBCG_PV_UNR
#define PBCG_PV_UNR 8
#endif
#ifndef PBCG_PV_MAXSTAGES
#define PBCG_PV_MAXSTAGES 8
#endif
#ifndef PBCG_PV_NCW_G
#define PBCG_PV_NCW_G 30
#endif
#ifndef PBCG_PV_UNR_G
#define PBCG_PV_UNR_G 3  // C4 SpMV (prefetched, 30 warps): 2: 280, 3: 251, 4: 264, 8 without prefetch: 299 us
#endif
#ifndef PBCG_PV_PF_G
#define PBCG_PV_PF_G 1
#endif
#ifndef PBCG_PV_MIN_WIN_STAGES
#define PBCG_PV_MIN_WIN_STAGES 6
#endif
static constexpr int PV_TMA_MAX_WINDOW = 48 * 1024;  // bytes of x window up to which the matrix rides the ring
static constexpr int PV_NCW = PBCG_PV_NCW, PV_CAP = PBCG_PV_CAP, PV_UNR = PBCG_PV_UNR,
                     PV_MAXSTAGES = PBCG_PV_MAXSTAGES, PV_MIN_WIN_STAGES = PBCG_PV_MIN_WIN_STAGES,
                     PV_NCW_G = PBCG_PV_NCW_G, PV_UNR_G = PBCG_PV_UNR_G;
static constexpr bool PV_PF_G = PBCG_PV_PF_G != 0;

struct Rank {
    int id = 0;
    int64_t rb = 0, re = 0, n = 0;
    int64_t buf_lo = 0, buf_hi = 0, own_off = 0;  // padded x-buffer covers global [buf_lo, buf_hi)
    std::vector<int64_t> recv_lo, recv_hi, send_lo, send_hi;
    int64_t nslices = 0, sell_nnz = 0;
    std::vector<int64_t> h_slice_off;
    // device
    int64_t *slice_off = nullptr;
    int32_t *row_len = nullptr;
    double *sval = nullptr;
    int32_t *scol = nullptr;
    double *x = nullptr, *r = nullptr, *rh = nullptr, *p = nullptr, *s = nullptr, *q = nullptr, *y = nullptr,
           *t = nullptr, *v = nullptr, *b = nullptr, *tmp = nullptr;
    double *zpad = nullptr, *wpad = nullptr, *xpad = nullptr;
    long long *gacc[NPH] = {};
    long long *gsm = nullptr;  // fused small-system kernel: phase buffers gA[2], gB[2] (GW4 words each)
    unsigned *gbar = nullptr;  // its grid barrier
    unsigned *tickets = nullptr;
    Scalars *sc = nullptr;
    double *hist = nullptr;
    int *bad = nullptr;
    double *z() const { return zpad + own_off; }
    double *w() const { return wpad + own_off; }
    std::vector<int32_t> h_perm;  // SELL position -> local row (empty: identity)
    int32_t max_len = 0;          // longest row of this rank
    int32_t *perm = nullptr;
    int32_t *slot_rec = nullptr;  // SELL_RS slot records per slice (SellMat::slot_rec)
    bool use_slots = true;
    int64_t nnz = 0, n_explicit = 0;  // stored nonzeros, column ids that stay explicit
    int spmv_kind = 0;                // SpMV kernel (set at setup)
    double *dg = nullptr;             // Jacobi: diag(A) of this rank's rows
    double *bjm = nullptr, *bji = nullptr;  // 2x2 block Jacobi: M and M^-1 of this rank's blocks (4 doubles each)
    // pipelined 2x2 block Jacobi (R-25): the SpMV inputs z_hat = M^-1 z and
    // w_hat = M^-1 w (padded like z, w; halo-exchanged instead of them)
    bool pipe = false;
    int64_t ng = 0;  // global order (block of the last row)
    double *zhpad = nullptr, *whpad = nullptr;
    double *part[NPH] = {};           // plain dot mode: CTA partials [PLAIN_GRID][4] per phase
    double *pdsum = nullptr;          // plain dot mode, NCCL ranks: local sums [NPH][4] (allreduced)
    // packed SELL-P chunks (rows <= 8 nonzeros) or SELL-V chunks (longer
    // rows): blob + byte offsets per chunk; h_cs: first slice of each SELL-V chunk
    int64_t nchunks = 0, blob_cap = 0, blob_bytes = 0;
    std::vector<int32_t> h_cs;
    int32_t *cxlo = nullptr, *cxhi = nullptr;  // SELL-V: x-buffer index range [lo, hi) of each chunk
    int ps_xr = 0;                             // SELL-V: x-window ring (doubles, a multiple of 64)
    bool pv_gld = false;                       // SELL-V: matrix loaded from global (only headers in the ring)
    unsigned char *blob = nullptr;
    int64_t *blob_off = nullptr;
    uint8_t *nexp = nullptr;
    int ps_stage = 0, ps_stages = 0;  // ring geometry of spmv_sellp_kernel (bytes per stage, stages)
    // multi-rank halo overlap: the interior units [in_lo, in_hi) (chunks for
    // the SELL-P kernel, slices otherwise) read no halo entry
    bool split = false;
    int64_t in_lo = 0, in_hi = 0;
    // chunked start (x0 = 0, host b, one rank; plan_start): row boundaries
    // st_row[0..NCH] of the chunks and the SpMV units st_u[0..NCH] covering
    // them; chunk k's rows read x rows of chunks <= k + 1 only
    std::vector<int64_t> st_row, st_u;
    SellMat mat(int64_t p0 = 0, int64_t p1 = -1) const {
        return SellMat{n, slice_off, row_len, sval, scol, h_perm.empty() ? nullptr : perm,
                       use_slots ? slot_rec : nullptr, p0, p1 < 0 ? n : std::min<int64_t>(p1, n)};
    }
};

struct pbcg_handle {
    int dev = 0, nsm = 148;
    cudaStream_t stream = nullptr, side = nullptr, cstream = nullptr;  // cstream: halo exchange (overlap)
    int nranks = 1, rank = 0, V = 1;  // real ranks, this rank, virtual ranks
    bool comm = false;                // NCCL communicators exist (nranks > 1, or forced for testing)
    int64_t n_global = 0;
    bool comm_only = false;
    int precond = PBCG_PRECOND_NONE;  // pbcg_dist.precond
    std::vector<Rank> R;
    ncclComm_t comm_halo = nullptr, comm_red = nullptr;
    long long **vgacc = nullptr;  // device array [NPH][V] of gacc pointers (virtual ranks)
    double **vpart = nullptr;     // device array [NPH][V] of plain-mode partial arrays
    int dot_mode = PBCG_DOT_EXACT;  // of the running solve (pbcg_opts.dot_mode)
    int method = PBCG_METHOD_PBICGSTAB;  // of the running solve (pbcg_opts.method)
    int rr_period = 0;                   // residual replacement period of the running solve (0: never)
    int64_t it_enq = 0;                  // iterations enqueued since start (host-side count)
    int g_mode[2] = {-1, -1};       // dot mode + 2 method each captured graph was built with
    int hist_cap = 10001;
    Scalars *h_sc = nullptr;      // pinned mirror of rank 0's scalars
    Scalars *h_poll[2] = {};      // pinned scalars copies of the last two solve chunks
    cudaEvent_t evp[2] = {};      // their copies done
    int grid_md = 0;
    int small_grid = 0;  // fused small-system kernel: cooperative grid (0: not eligible)
    // captured iteration graphs: [0] one chunk of `chunk` iterations, [1] the
    // last remainder length (iterate(k) = k / chunk replays of [0] + one of [1])
    cudaGraphExec_t gexec[2] = {nullptr, nullptr};
    int g_iters[2] = {0, 0};
    int chunk = 16;                 // iterations per graph chunk (pbcg_opts.poll_every of the last start)
    cudaEvent_t ev[8] = {};
    cudaEvent_t evh[4] = {};  // halo-overlap fork/join (multi-rank)
    cudaEvent_t evc[16] = {};  // start: chunks of the host copy of b landed (START_NCH)
    cudaEvent_t t0 = nullptr, t1 = nullptr;
    bool started = false;
    int max_iter = 0;
    size_t ws_need = 0;
    // scratch for exdot on a handle
    double *xd_out = nullptr;
    int32_t *xd_flags = nullptr;
};

static constexpr int64_t SELL_SIGMA = 256;  // sorting window (rows) for irregular matrices

// workspace carving (dry run computes the size)
struct Carver {
    char *base;
    size_t off = 0;
    template <class T>
    T *take(size_t count) {
        off = (off + 255) & ~size_t(255);
        T *p = base ? (T *)(base + off) : nullptr;
        off += std::max<size_t>(count, 1) * sizeof(T);
        return p;
    }
};

static void carve_rank(Carver &C, Rank &R, int hist_cap, bool comm_only, int precond) {
    if (!comm_only) {
        R.slice_off = C.take<int64_t>(R.nslices + 16);      // + tail read by the TMA SpMV
        R.row_len = C.take<int32_t>((size_t)R.nslices * 32);  // whole slices, zero past n
        R.sval = C.take<double>(R.sell_nnz);
        R.scol = C.take<int32_t>(R.sell_nnz);
        R.slot_rec = C.take<int32_t>((size_t)R.nslices * SELL_RS);
        if (R.max_len <= 8) {  // SELL-P blob: worst case every slot explicit
            R.nchunks = (R.nslices + PS_SPS - 1) / PS_SPS;
            R.blob_cap = R.nchunks * (int64_t)(SellPGeo<PS_SPS>::H + 16) + 12 * R.sell_nnz;
            R.blob = C.take<unsigned char>((size_t)R.blob_cap);
            R.blob_off = C.take<int64_t>((size_t)R.nchunks + 1);
            R.nexp = C.take<uint8_t>((size_t)R.nslices);
        } else if (R.max_len <= 255) {  // SELL-V blob: every nonzero once + per-chunk headers
            R.blob_cap = 12 * R.nnz + 96 * R.nslices + 256 + 2048;  // + header-copy slack past the last chunk
            R.blob = C.take<unsigned char>((size_t)R.blob_cap);
            R.blob_off = C.take<int64_t>((size_t)R.nslices + 1);
            R.cxlo = C.take<int32_t>((size_t)R.nslices);
            R.cxhi = C.take<int32_t>((size_t)R.nslices);
        }
        R.perm = C.take<int32_t>(R.h_perm.size());
        const size_t n = (size_t)R.n + 2;
        R.x = C.take<double>(n); R.r = C.take<double>(n); R.rh = C.take<double>(n); R.p = C.take<double>(n);
        R.s = C.take<double>(n); R.q = C.take<double>(n); R.y = C.take<double>(n); R.t = C.take<double>(n);
        R.v = C.take<double>(n); R.b = C.take<double>(n); R.tmp = C.take<double>(n);
        const size_t nb = (size_t)(R.buf_hi - R.buf_lo) + 2;
        R.zpad = C.take<double>(nb); R.wpad = C.take<double>(nb); R.xpad = C.take<double>(nb);
        R.hist = C.take<double>((size_t)hist_cap * H_COLS);
        if (precond == PBCG_PRECOND_JACOBI) R.dg = C.take<double>((size_t)R.n + 2);
        if (precond == PBCG_PRECOND_BJACOBI2 || precond == PBCG_PRECOND_BJACOBI2_PIPE) {
            R.bjm = C.take<double>(4 * (size_t)((R.n + 1) / 2 + 1));
            R.bji = C.take<double>(4 * (size_t)((R.n + 1) / 2 + 1));
        }
        if (precond == PBCG_PRECOND_BJACOBI2_PIPE) {
            R.zhpad = C.take<double>(nb);
            R.whpad = C.take<double>(nb);
        }
    }
    for (int k = 0; k < NPH; ++k) R.gacc[k] = C.take<long long>(GW4);
    for (int k = 0; k < NPH; ++k) R.part[k] = C.take<double>((size_t)PLAIN_GRID * 4);
    R.pdsum = C.take<double>((size_t)NPH * 4);
    R.tickets = C.take<unsigned>(16);
    R.gsm = C.take<long long>(4 * (size_t)GW4);  // fused small-system kernel: gA[2], gB[2]
    R.gbar = C.take<unsigned>(16);
    R.sc = C.take<Scalars>(1);
    R.bad = C.take<int>(4);
}

static size_t carve_handle_extra(Carver &C, pbcg_handle *h) {
    h->vgacc = C.take<long long *>((size_t)NPH * h->V);
    h->vpart = C.take<double *>((size_t)NPH * h->V);
    h->xd_out = C.take<double>(4);
    h->xd_flags = C.take<int32_t>(4);
    return C.off;
}

// Plan ranks: row ranges, hulls, halo, slices.  h_rp: host row_ptr of the rows
// passed in (full matrix for virtual ranks).  hulls: 2 per rank (min,max col).
static int plan_ranks(pbcg_handle *h, const pbcg_csr_local *A, const std::vector<int32_t> &h_rp,
                      const std::vector<long long> &hulls, const std::vector<int64_t> &all_ranges) {
    const int P = h->V > 1 ? h->V : 1;
    h->R.assign(P, Rank());
    std::vector<int64_t> begins(P + 1);
    if (h->V > 1) pbcg_plan_partition(A->n_global, P, begins.data());
    else { begins[0] = A->row_begin; begins[1] = A->row_end; }
    // ranges of every (virtual or real) rank
    const int PR = h->V > 1 ? P : h->nranks;
    std::vector<int64_t> ranges(4 * PR);
    if (h->V > 1) {
        for (int v = 0; v < P; ++v) {
            ranges[4 * v] = begins[v];
            ranges[4 * v + 1] = begins[v + 1];
            ranges[4 * v + 2] = hulls[2 * v];
            ranges[4 * v + 3] = hulls[2 * v + 1];
        }
    } else {
        ranges = all_ranges;
    }
    for (int v = 0; v < P; ++v) {
        Rank &R = h->R[v];
        const int me = h->V > 1 ? v : h->rank;
        R.id = me;
        R.rb = begins[v];
        R.re = begins[v + 1];
        R.n = R.re - R.rb;
        R.recv_lo.resize(PR); R.recv_hi.resize(PR); R.send_lo.resize(PR); R.send_hi.resize(PR);
        int64_t blo, bhi;
        RC_TRY(pbcg_plan_halo(PR, me, ranges.data(), R.recv_lo.data(), R.recv_hi.data(), R.send_lo.data(),
                              R.send_hi.data(), &blo, &bhi));
        // align so that the owned part starts on a 32-byte boundary
        const int64_t lead = R.rb - blo;
        const int64_t lead_al = (lead + 3) & ~int64_t(3);
        R.buf_lo = R.rb - lead_al;
        R.buf_hi = bhi;
        R.own_off = lead_al;
        // sliced ELL: 32 rows per slice, width = longest row of the slice
        R.nslices = (R.n + 31) / 32;
        const int64_t r0 = (h->V > 1) ? R.rb : 0;  // index into h_rp
        auto rowlen = [&](int64_t r) { return h_rp[r0 + r + 1] - h_rp[r0 + r]; };
        auto slices = [&](const int32_t *perm) {
            R.h_slice_off.assign(R.nslices + 1, 0);
            for (int64_t sl = 0; sl < R.nslices; ++sl) {
                int32_t wmax = 0;
                const int64_t a = sl * 32, e = std::min<int64_t>(a + 32, R.n);
                for (int64_t q = a; q < e; ++q) wmax = std::max(wmax, rowlen(perm ? perm[q] : q));
                R.h_slice_off[sl + 1] = R.h_slice_off[sl] + 32 * (int64_t)wmax;
            }
            R.sell_nnz = R.h_slice_off[R.nslices];
        };
        slices(nullptr);
        R.max_len = 0;
        for (int64_t q = 0; q < R.n; ++q) R.max_len = std::max(R.max_len, rowlen(q));
        const int64_t nnz = (int64_t)h_rp[r0 + R.n] - h_rp[r0];
        R.nnz = nnz;
        R.h_perm.clear();
        if (R.sell_nnz > nnz + nnz / 16) {
            // sigma-sorting (sliced ELL-C-sigma, C = 32, sigma = SELL_SIGMA): rows
            // of each window sorted by length so that a slice holds rows of
            // similar length -- the per-row summation order is unchanged
            R.h_perm.resize(R.n);
            for (int64_t q = 0; q < R.n; ++q) R.h_perm[q] = (int32_t)q;
            for (int64_t w0 = 0; w0 < R.n; w0 += SELL_SIGMA) {
                const int64_t w1 = std::min<int64_t>(w0 + SELL_SIGMA, R.n);
                std::stable_sort(R.h_perm.begin() + w0, R.h_perm.begin() + w1,
                                 [&](int32_t a, int32_t b) { return rowlen(a) > rowlen(b); });
            }
            slices(R.h_perm.data());
        }
    }
    return PBCG_OK;
}

static int compute_hulls(const pbcg_csr_local *A, int P, const std::vector<int64_t> &begins_local,
                         std::vector<long long> &hulls) {
    const int64_t nloc = A->row_end - A->row_begin;
    hulls.assign(2 * P, 0);
    for (int v = 0; v < P; ++v) { hulls[2 * v] = INT64_MAX; hulls[2 * v + 1] = INT64_MIN; }
    if (nloc == 0) return PBCG_OK;
    long long *d_h = nullptr;
    CUDA_TRY(cudaMalloc(&d_h, sizeof(long long) * 2 * P));
    CUDA_TRY(cudaMemcpy(d_h, hulls.data(), sizeof(long long) * 2 * P, cudaMemcpyHostToDevice));
    for (int v = 0; v < P; ++v) {
        const int64_t rows = begins_local[v + 1] - begins_local[v];
        if (rows <= 0) continue;
        const int grid = (int)std::min<int64_t>((rows + 255) / 256, 1184);
        row_hull_kernel<<<grid, 256>>>(begins_local[v], begins_local[v + 1], A->row_ptr, A->col_idx, d_h + 2 * v);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaMemcpy(hulls.data(), d_h, sizeof(long long) * 2 * P, cudaMemcpyDeviceToHost));
    cudaFree(d_h);
    return PBCG_OK;
}

static int validate_csr(const pbcg_csr_local *A, const pbcg_dist *d) {
    if (!A) return PBCG_OK;
    if (A->n_global < 1 || A->row_begin < 0 || A->row_end < A->row_begin || A->row_end > A->n_global)
        return fail(PBCG_EINVAL, "csr: bad dimensions (n=%lld rows [%lld,%lld))", (long long)A->n_global,
                    (long long)A->row_begin, (long long)A->row_end);
    if (A->n_global > INT32_MAX) return fail(PBCG_EINVAL, "csr: n_global exceeds int32 column ids");
    if ((A->row_end > A->row_begin) && (!A->row_ptr || (A->nnz_local > 0 && (!A->col_idx || !A->values))))
        return fail(PBCG_EINVAL, "csr: null array");
    if (d && d->virtual_ranks > 1 && (A->row_begin != 0 || A->row_end != A->n_global))
        return fail(PBCG_EINVAL, "virtual ranks need the full matrix");
    return PBCG_OK;
}

// Everything workspace_size and setup share: host row_ptr, hulls, plan.
static int prepare(pbcg_handle *h, const pbcg_csr_local *A, const pbcg_dist *d, std::vector<int32_t> &h_rp,
                   const std::vector<int64_t> *all_ranges) {
    h->nranks = d ? std::max(1, d->nranks) : 1;
    h->rank = d ? d->rank : 0;
    h->V = (d && d->virtual_ranks > 1) ? d->virtual_ranks : 1;
    h->hist_cap = (d && d->history_capacity > 0) ? d->history_capacity : 10001;
    h->precond = d ? d->precond : PBCG_PRECOND_NONE;
    if (h->precond != PBCG_PRECOND_NONE && h->precond != PBCG_PRECOND_JACOBI && h->precond != PBCG_PRECOND_BJACOBI2 &&
        h->precond != PBCG_PRECOND_BJACOBI2_PIPE)
        return fail(PBCG_EINVAL, "bad precond");
    if (h->nranks > 1 && h->V > 1) return fail(PBCG_EINVAL, "virtual ranks need nranks == 1");
    if (h->rank < 0 || h->rank >= h->nranks) return fail(PBCG_EINVAL, "bad rank");
    if (!A) {
        h->comm_only = true;
        h->R.assign(h->V, Rank());
        return PBCG_OK;
    }
    RC_TRY(validate_csr(A, d));
    h->n_global = A->n_global;
    const int64_t nloc = A->row_end - A->row_begin;
    if (h->V > nloc) return fail(PBCG_EINVAL, "more virtual ranks than rows");
    h_rp.resize(nloc + 1);
    CUDA_TRY(cudaMemcpy(h_rp.data(), A->row_ptr, sizeof(int32_t) * (nloc + 1), cudaMemcpyDeviceToHost));
    if (h_rp[0] != 0) return fail(PBCG_EINVAL, "csr: row_ptr[0] != 0");
    for (int64_t r = 0; r < nloc; ++r)
        if (h_rp[r + 1] < h_rp[r]) return fail(PBCG_EINVAL, "csr: row_ptr decreases at row %lld", (long long)r);
    if (h_rp[nloc] != A->nnz_local) return fail(PBCG_EINVAL, "csr: nnz_local != row_ptr[n]");
    const int P = h->V;
    std::vector<int64_t> begins(P + 1);
    if (P > 1) pbcg_plan_partition(nloc, P, begins.data());
    else { begins[0] = 0; begins[1] = nloc; }
    std::vector<long long> hulls;
    RC_TRY(compute_hulls(A, P, begins, hulls));
    std::vector<int64_t> ranges;
    if (h->V == 1) {
        if (all_ranges) ranges = *all_ranges;
        else ranges = {A->row_begin, A->row_end, hulls[0], hulls[1]};  // local-only view (size query)
    }
    if (h->V == 1 && !all_ranges) {
        // size query for one real rank: the buffer hull only depends on local rows
        h->nranks = 1;
        h->rank = 0;
    }
    return plan_ranks(h, A, h_rp, hulls, ranges);
}

static size_t total_size(pbcg_handle *h) {
    Carver C{nullptr};
    for (auto &R : h->R) carve_rank(C, R, h->hist_cap, h->comm_only, h->precond);
    return carve_handle_extra(C, h) + 256;
}

// 2x2 block Jacobi (R-23): the CSR of B's pattern (every column block a row
// touches contributes both its columns; A's values there, +0.0 at the added
// ones) in device memory owned by `own` (freed by its destructor), used in
// place of A for the layout; B's values are formed after the SELL is built.
struct BjCsr {
    pbcg_csr_local B{};
    int32_t *rp = nullptr, *col = nullptr;
    double *val = nullptr;
    ~BjCsr() { cudaFree(rp); cudaFree(col); cudaFree(val); }
};
static int bj_expand(const pbcg_csr_local *A, BjCsr &o) {
    const int64_t nloc = A->row_end - A->row_begin;
    if (nloc <= 0) { o.B = *A; return PBCG_OK; }
    CUDA_TRY(cudaMalloc(&o.rp, sizeof(int32_t) * (nloc + 1)));
    const int g = (int)std::min<int64_t>((nloc + 255) / 256, 65535);
    bj_count_kernel<<<g, 256>>>(nloc, A->row_ptr, A->col_idx, A->n_global, o.rp + 1);
    CUDA_TRY(cudaGetLastError());
    std::vector<int32_t> cnt(nloc + 1, 0);
    CUDA_TRY(cudaMemcpy(cnt.data() + 1, o.rp + 1, sizeof(int32_t) * nloc, cudaMemcpyDeviceToHost));
    int64_t tot = 0;
    for (int64_t r = 1; r <= nloc; ++r) {
        tot += cnt[r];
        if (tot > INT32_MAX) return fail(PBCG_EINVAL, "block jacobi: expanded matrix exceeds 2^31 entries");
        cnt[r] = (int32_t)tot;
    }
    CUDA_TRY(cudaMemcpy(o.rp, cnt.data(), sizeof(int32_t) * (nloc + 1), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc(&o.col, sizeof(int32_t) * std::max<int64_t>(tot, 1)));
    CUDA_TRY(cudaMalloc(&o.val, sizeof(double) * std::max<int64_t>(tot, 1)));
    bj_fill_kernel<<<g, 256>>>(nloc, A->row_ptr, A->col_idx, A->values, A->n_global, o.rp, o.col, o.val);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    o.B = *A;
    o.B.nnz_local = tot;
    o.B.row_ptr = o.rp;
    o.B.col_idx = o.col;
    o.B.values = o.val;
    return PBCG_OK;
}

extern "C" int pbicgstab_workspace_size(const pbcg_csr_local *A, const pbcg_dist *d, size_t *bytes) {
    if (!bytes) return fail(PBCG_EINVAL, "bytes == NULL");
    pbcg_handle tmp;
    std::vector<int32_t> h_rp;
    BjCsr bj;
    if (A && d && d->precond == PBCG_PRECOND_BJACOBI2) {
        RC_TRY(validate_csr(A, d));
        RC_TRY(bj_expand(A, bj));
        A = &bj.B;
    }
    RC_TRY(prepare(&tmp, A, d, h_rp, nullptr));
    *bytes = total_size(&tmp);
    return PBCG_OK;
}

static int grid_for(const void *kern, int bs, int nsm, size_t smem = 0) {
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, bs, smem) != cudaSuccess || occ < 1) occ = 1;
    return occ * nsm;
}

// ----------------------------------------------------------------------------
// halo exchange and cross-rank reduction
// ----------------------------------------------------------------------------
// padded buffer selector: 0 = z, 1 = w, 2 = x scratch
// (pipelined block Jacobi: the SpMV inputs are z_hat, w_hat; z, w stay own-only)
static double *padbuf(Rank &R, int which) {
    return which == 0 ? (R.pipe ? R.zhpad : R.zpad) : which == 1 ? (R.pipe ? R.whpad : R.wpad) : R.xpad;
}

static int halo(pbcg_handle *h, int which, cudaStream_t st = nullptr) {
    if (!st) st = h->stream;
    const int P = (int)h->R.size();
    if (h->V > 1) {
        for (int me = 0; me < P; ++me) {
            Rank &R = h->R[me];
            for (int q = 0; q < P; ++q) {
                const int64_t lo = R.recv_lo[q], hi = R.recv_hi[q];
                if (hi <= lo) continue;
                Rank &Q = h->R[q];
                CUDA_TRY(cudaMemcpyAsync(padbuf(R, which) + (lo - R.buf_lo), padbuf(Q, which) + (lo - Q.buf_lo),
                                         sizeof(double) * (hi - lo), cudaMemcpyDeviceToDevice, st));
            }
        }
        return PBCG_OK;
    }
    if (!h->comm) return PBCG_OK;
    Rank &R = h->R[0];
    NCCL_TRY(g_nccl.GroupStart());
    for (int q = 0; q < h->nranks; ++q) {
        if (R.send_hi[q] > R.send_lo[q])
            NCCL_TRY(g_nccl.Send(padbuf(R, which) + (R.send_lo[q] - R.buf_lo), (size_t)(R.send_hi[q] - R.send_lo[q]),
                                 ncclFloat64, q, h->comm_halo, st));
        if (R.recv_hi[q] > R.recv_lo[q])
            NCCL_TRY(g_nccl.Recv(padbuf(R, which) + (R.recv_lo[q] - R.buf_lo), (size_t)(R.recv_hi[q] - R.recv_lo[q]),
                                 ncclFloat64, q, h->comm_halo, st));
    }
    NCCL_TRY(g_nccl.GroupEnd());
    return PBCG_OK;
}

// sum the phase-`ph` superaccumulators over ranks, then round + finalise
template <int ND>
static int reduce_finalize(pbcg_handle *h, int ph, int phase, cudaStream_t st, double *out, int32_t *oflags) {
    NvtxRange nvtx_("pbcg.allreduce+finalize");
    if (h->dot_mode == PBCG_DOT_PLAIN && (phase == PH_A || phase == PH_B)) {
        // plain dots: every rank sums all partials in the same order (virtual
        // ranks), or its own and then an fp64 allreduce (NCCL: order chosen by NCCL)
        for (auto &R : h->R) {
            if (h->comm) {
                plain_finalize_kernel<ND><<<1, 32, 0, st>>>(h->vpart + (size_t)ph * h->V, 1, h->nsm, phase, R.sc,
                                                           R.hist, R.pdsum + 4 * ph, 0);
                CUDA_TRY(cudaGetLastError());
                NCCL_TRY(g_nccl.AllReduce(R.pdsum + 4 * ph, R.pdsum + 4 * ph, ND, ncclFloat64, ncclSum, h->comm_red, st));
                plain_phase_kernel<<<1, 32, 0, st>>>(phase, R.sc, R.pdsum + 4 * ph, R.hist);
            } else {
                plain_finalize_kernel<ND><<<1, 32, 0, st>>>(h->vpart + (size_t)ph * h->V, h->V, h->nsm, phase, R.sc,
                                                           R.hist, nullptr, 1);
            }
            CUDA_TRY(cudaGetLastError());
        }
        return PBCG_OK;
    }
    const int words = xs_words(ND);  // fast words, flag counts and the extended words (R-24)
    if (h->V > 1) {
        vallreduce_kernel<<<(words + 127) / 128, 128, 0, st>>>(h->vgacc + (size_t)ph * h->V, h->V, words);
        CUDA_TRY(cudaGetLastError());
    } else if (h->comm) {
        NCCL_TRY(g_nccl.AllReduce(h->R[0].gacc[ph], h->R[0].gacc[ph], (size_t)words, ncclInt64, ncclSum, h->comm_red, st));
    }
    for (auto &R : h->R) {
        finalize_kernel<ND><<<1, 128, 0, st>>>(R.gacc[ph], phase, R.sc, R.hist, out, oflags);
        CUDA_TRY(cudaGetLastError());
        out = nullptr;  // only the first (virtual) rank writes the exdot result
        oflags = nullptr;
    }
    return PBCG_OK;
}

static bool multi(const pbcg_handle *h) { return h->V > 1 || h->comm; }


// SpMV kernel choice.  Short rows (every row <= 8 nonzeros: stencils) and
// at least SELLP_MIN_SLICES_PER_SM slices per SM: the TMA kernel on the packed
// SELL-P chunks (spmv_sellp_kernel); smaller short-row matrices: the
// register-pipelined persistent kernel (no ring to fill); long rows: one row
// per thread (more warps in flight).  PBCG_SPMV_KERNEL=tma|pipe|plain
// overrides (A/B runs).
enum { SPMV_K_PLAIN = 0, SPMV_K_PIPE = 1, SPMV_K_TMA = 2, SPMV_K_TMAV = 3 };
static constexpr int SPMV_COMM_SMS = 4;  // SMs the interior SpMV leaves to the halo's NCCL kernels
static constexpr int64_t SELLP_MIN_SLICES_PER_SM = 32;  // C3 (443/SM): TMA 7.17K vs 6.18K iter/s; C1 (1/SM): pipe
static constexpr int64_t SELLV_MIN_SLICES_PER_SM = 16;
static int spmv_kind_for(const Rank &R, int nsm) {  // at setup
    const char *e = getenv("PBCG_SPMV_KERNEL");
    if (R.max_len > 8) {  // long rows: the SELL-V kernel (rows <= 255 nonzeros), else one row per thread
        const bool v_ok = R.max_len <= 255 && R.blob;
        if (e) return v_ok && (strcmp(e, "tma") == 0 || strcmp(e, "tmav") == 0) ? SPMV_K_TMAV : SPMV_K_PLAIN;
        return v_ok && R.nslices >= SELLV_MIN_SLICES_PER_SM * nsm ? SPMV_K_TMAV : SPMV_K_PLAIN;
    }
    if (!e) return R.nslices >= SELLP_MIN_SLICES_PER_SM * nsm ? SPMV_K_TMA : SPMV_K_PIPE;
    return strcmp(e, "pipe") == 0 ? SPMV_K_PIPE : strcmp(e, "tma") == 0 ? SPMV_K_TMA : SPMV_K_PLAIN;
}

// Launch with programmatic stream serialisation (PDL): the iteration kernels
// call pdl_sync() after their prologue, so their launch and prologue overlap
// the previous kernel's tail.  PBCG_PDL=0 turns it off (A/B runs).
static int g_pdl = -1;
static bool pdl_on() {
    if (g_pdl < 0) {
        const char *e = getenv("PBCG_PDL");
        g_pdl = (e && e[0] == '0') ? 0 : 1;
    }
    return g_pdl == 1;
}
// PDL only where every kernel of the iteration is persistent (one CTA per SM):
// with the many-wave row-per-thread SpMV (long rows, C4) the early launches
// cost 10 % (1316 -> 1199 iter/s), so that path launches without it.
static bool pdl_for(const Rank &R);
template <typename... KArgs, typename... Args>
static void launch_ex(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                      Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = (pdl && pdl_on()) ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, args...);  // errors surface in the caller's cudaGetLastError
}

static bool pdl_for(const Rank &R) { return R.spmv_kind != SPMV_K_PLAIN; }

// units [u0, u1): chunks for the SELL-P kernel, slices otherwise (u1 < 0: all);
// reserve: SMs left free (the halo exchange's NCCL kernels during overlap)
template <int MODE>
static void spmv_dispatch(pbcg_handle *h, const Rank &R, const double *xpad, double *y, const double *b, double *y2,
                          const Scalars *sc, cudaStream_t st, int64_t u0, int64_t u1, int reserve) {
    if (R.spmv_kind == SPMV_K_TMA) {
        if (u1 < 0) u1 = R.nchunks;
        auto *k = spmv_sellp_kernel<MODE, PS_SPS, PS_RPW>;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute((const void *)k, cudaFuncAttributeMaxDynamicSharedMemorySize, PS_SMEM_MAX);
            attr = true;
        }
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->nsm - reserve, u1 - u0));
        const size_t smem = (size_t)R.ps_stages * R.ps_stage + 2 * R.ps_stages * sizeof(uint64_t);
        launch_ex(k, dim3(grid), dim3((PS_SPS / PS_RPW + 1) * 32), smem, st, pdl_for(R), R.n, R.nslices,
                  (const unsigned char *)R.blob, (const int64_t *)R.blob_off,
                  (const int32_t *)(R.h_perm.empty() ? nullptr : R.perm), xpad, y, b, y2, sc, R.ps_stage, R.ps_stages,
                  u0, u1);
        return;
    }
    if (R.spmv_kind == SPMV_K_TMAV) {
        if (u1 < 0) u1 = R.nchunks;
        auto *k = R.pv_gld ? spmv_sellv_kernel<MODE, PV_NCW_G, PV_UNR_G, true, PV_PF_G>
                           : spmv_sellv_kernel<MODE, PV_NCW, PV_UNR, false>;
        static bool attr = false;
        if (!attr) {
            cudaFuncSetAttribute((const void *)spmv_sellv_kernel<MODE, PV_NCW_G, PV_UNR_G, true, PV_PF_G>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, PS_SMEM_MAX);
            cudaFuncSetAttribute((const void *)spmv_sellv_kernel<MODE, PV_NCW, PV_UNR, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, PS_SMEM_MAX);
            attr = true;
        }
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->nsm - reserve, u1 - u0));
        const size_t smem = (size_t)R.ps_stages * R.ps_stage + 8 * (size_t)R.ps_xr + 2 * R.ps_stages * sizeof(uint64_t);
        launch_ex(k, dim3(grid), dim3(((R.pv_gld ? PV_NCW_G : PV_NCW) + 1) * 32), smem, st, pdl_for(R), R.n,
                  (const unsigned char *)R.blob,
                  (const int64_t *)R.blob_off, (const int32_t *)R.cxlo, (const int32_t *)R.cxhi,
                  (const int32_t *)(R.h_perm.empty() ? nullptr : R.perm), xpad, y, b, y2, sc, R.ps_stage, R.ps_stages,
                  R.ps_xr, u0, u1);
        return;
    }
    if (u1 < 0) u1 = R.nslices;
    const SellMat M = R.mat(u0 * 32, u1 * 32);
    const int64_t rows = M.p1 - M.p0;
    if (rows <= 0) return;
    if (R.spmv_kind == SPMV_K_PIPE) {
        static int per_sm = 0;
        if (!per_sm) per_sm = std::max(1, grid_for((const void *)spmv_sell_pipe_kernel<MODE, 8>, 256, 1));
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)per_sm * (h->nsm - reserve), (rows + 255) / 256));
        launch_ex(spmv_sell_pipe_kernel<MODE, 8>, dim3(grid), dim3(256), 0, st, pdl_for(R), M, xpad, y, b, y2, sc);
    } else {
        const int grid = (int)((rows + 255) / 256);
#ifndef PBCG_PLAIN_UNR
#define PBCG_PLAIN_UNR 8
#endif
        launch_ex(spmv_sell_kernel<MODE, PBCG_PLAIN_UNR, 1>, dim3(grid), dim3(256), 0, st, false, M, xpad, y, b, y2,
                  sc);
    }
}

// part: 0 = all rows, 1 = the interior (no halo entries), 2 = the boundary
enum { SP_ALL = 0, SP_INTERIOR = 1, SP_BOUNDARY = 2 };
static int launch_spmv(pbcg_handle *h, Rank &R, int mode, const double *xpad, double *y, const double *b, double *y2,
                       bool predicated, cudaStream_t st, int part = SP_ALL, int reserve = 0) {
    if (R.n == 0) return PBCG_OK;
    const Scalars *sc = predicated ? R.sc : nullptr;
    auto go = [&](int64_t u0, int64_t u1, int rsv) {
        if (u1 >= 0 && u1 <= u0) return;
        if (mode == SPMV_PLAIN) spmv_dispatch<SPMV_PLAIN>(h, R, xpad, y, b, y2, sc, st, u0, u1, rsv);
        else spmv_dispatch<SPMV_RESID>(h, R, xpad, y, b, y2, sc, st, u0, u1, rsv);
    };
    if (part == SP_ALL || !R.split) {
        go(0, -1, 0);
    } else if (part == SP_INTERIOR) {
        go(R.in_lo, R.in_hi, reserve);
    } else {
        const int64_t units = (R.spmv_kind == SPMV_K_TMA || R.spmv_kind == SPMV_K_TMAV) ? R.nchunks : R.nslices;
        go(0, R.in_lo, 0);
        go(R.in_hi, units, 0);
    }
    CUDA_TRY(cudaGetLastError());
    return PBCG_OK;
}

// up-to-4 fused EXDOTs over every rank's rows (phase PH_INIT / PH_TRUE)
static int launch_xd1(pbcg_handle *h, const MultiDotArgs &a);
static int launch_xd2(pbcg_handle *h, const MultiDotArgs &a);

static int multidot(pbcg_handle *h, int ph, int phase, int nd, const double *const *xs_per_rank[4],
                    const double *const *ys_per_rank[4]) {
    const bool fin = !multi(h);
    for (size_t v = 0; v < h->R.size(); ++v) {
        Rank &R = h->R[v];
        MultiDotArgs a{};
        a.n = R.n;
        for (int d = 0; d < 4; ++d) {
            a.x[d] = d < nd ? xs_per_rank[d][v] : nullptr;
            a.y[d] = d < nd ? ys_per_rank[d][v] : nullptr;
        }
        a.sc = R.sc;
        a.gacc = R.gacc[ph];
        a.ticket = R.tickets + ph;
        a.hist = R.hist;
        a.phase = phase;
        a.finalize = fin;
        const int grid = std::max(1, std::min<int>(h->grid_md, (int)((R.n / 2 + K_BS - 1) / K_BS)));
        const bool aligned = ((((uintptr_t)a.x[0]) | ((uintptr_t)a.y[0])) & 15) == 0;
        if (nd == 1 && R.n > 0 && aligned) {
            RC_TRY(launch_xd1(h, a));  // one dot over aligned vectors: the TMA-streamed EXDOT kernel
        } else if (nd == 2 && R.n > 0 && aligned && a.x[1] == a.y[0] && a.y[1] == a.y[0]) {
            RC_TRY(launch_xd2(h, a));  // (x,y), (y,y): the two-dot stream kernel
        } else if (nd == 4) multidot_kernel<4, K_NP, K_NE, K_BS, U_MD4><<<grid, K_BS, 0, h->stream>>>(a);
        else if (nd == 2) multidot_kernel<2, K_NP, K_NE, K_BS, U_MD4><<<grid, K_BS, 0, h->stream>>>(a);
        else multidot_kernel<1, K_NP, K_NE, K_BS, U_MD1><<<grid, K_BS, 0, h->stream>>>(a);
        CUDA_TRY(cudaGetLastError());
    }
    if (!fin) {
        if (nd == 4) RC_TRY(reduce_finalize<4>(h, ph, phase, h->stream, nullptr, nullptr));
        else if (nd == 2) RC_TRY(reduce_finalize<2>(h, ph, phase, h->stream, nullptr, nullptr));
        else RC_TRY(reduce_finalize<1>(h, ph, phase, h->stream, nullptr, nullptr));
    }
    return PBCG_OK;
}

// ----------------------------------------------------------------------------
// one iteration of Algorithm 2 (enqueue only)
// ----------------------------------------------------------------------------
// Streaming (TMA-pipelined) kernel geometry -- performance parameters only.
// FPE levels (performance parameters only, R-16): hot p / hot e / cold, per
// kernel.  Chosen on C3/C4/C5 (profiles/r01): the p stream of the solver
// vectors spills more than the e stream, K3's cold levels rarely overflow.
#ifndef PBCG_K2_FPE
#define PBCG_K2_FPE 3, K2_NHE = 2, K2_NC = 3
#endif
#ifndef PBCG_K3_FPE
#define PBCG_K3_FPE 3, K3_NHE = 2, K3_NC = 2
#endif
static constexpr int K2_NH = PBCG_K2_FPE;
static constexpr int K3_NH = PBCG_K3_FPE;
#ifndef PBCG_S_NCW
#define PBCG_S_NCW 7
#endif
static constexpr int S_NCW = PBCG_S_NCW;  // K2: warps per dot group (2*7+1 = 15 warps per CTA)
#ifndef PBCG_K3_NCW
#define PBCG_K3_NCW 8  // C5 K3 241 -> 228 us vs 7 warps per group (9: 238, 10: spills)
#endif
static constexpr int K3_NCW = PBCG_K3_NCW;  // K3: warps per dot group (3 dots: fewer registers than K2)
#ifndef PBCG_X_NCW
#define PBCG_X_NCW 12
#endif
static constexpr int X_NCW = PBCG_X_NCW;
#ifndef PBCG_X_NH
#define PBCG_X_NH 2
#endif
#ifndef PBCG_X_NL
#define PBCG_X_NL 2
#endif
static constexpr int X_NH = PBCG_X_NH, X_NL = PBCG_X_NL;  // standalone EXDOT: hot / cold levels
#ifndef PBCG_K2_PPT
#define PBCG_K2_PPT 1
#endif
#ifndef PBCG_K2_ST
#define PBCG_K2_ST 5
#endif
#ifndef PBCG_K3_PPT
#define PBCG_K3_PPT 1
#endif
#ifndef PBCG_K3_ST
#define PBCG_K3_ST 5
#endif
#ifndef PBCG_XD_PPT
#define PBCG_XD_PPT 6
#endif
#ifndef PBCG_XD_ST
#define PBCG_XD_ST 2
#endif
static constexpr int K2_PPT = PBCG_K2_PPT, K2_ST = PBCG_K2_ST, K3_PPT = PBCG_K3_PPT, K3_ST = PBCG_K3_ST,
                     XD_PPT = PBCG_XD_PPT, XD_ST = PBCG_XD_ST;
#define K2S k2_stream<K2_NH, K2_NC, S_NCW, K2_PPT, K2_ST, K2_NHE>
#define K3S k3_stream<K3_NH, K3_NC, K3_NCW, K3_PPT, K3_ST, K3_NHE>
// lean variants (one cold level less and, round 3, one hot p level less):
// less end-of-kernel drain and a shorter hot cascade, which is what counts
// below LEAN_ROWS rows per rank (C1/C3/C4 measured faster, C5 slower).
// Hot p levels 3 -> 2 in the lean K2 / K3 (tools/ab_iter.py, iter/s): C3
// 7,504 -> 7,598 / 7,595 each, C4 1,552 -> 1,559 / 1,558; on C5 (not lean)
// the same change loses 2.2 % / 0.8 %.
#ifndef PBCG_LEAN_NH
#define PBCG_LEAN_NH 2
#endif
#ifndef PBCG_K2L_NCW
#define PBCG_K2L_NCW 7
#endif
#ifndef PBCG_K3L_NCW
#define PBCG_K3L_NCW 8
#endif
static constexpr int K2L_NCW = PBCG_K2L_NCW, K3L_NCW = PBCG_K3L_NCW;  // lean: warps per dot group
#define K2SL k2_stream<PBCG_LEAN_NH, K2_NC - 1, K2L_NCW, K2_PPT, K2_ST, K2_NHE>
#define K3SL k3_stream<PBCG_LEAN_NH, K3_NC - 1, K3L_NCW, K3_PPT, K3_ST, K3_NHE>
static constexpr int64_t LEAN_ROWS = 8 << 20;
#define K2SP k2_stream<K2_NH, K2_NC, S_NCW, K2_PPT, K2_ST, K2_NHE, false>
#define K3SP k3_stream<K3_NH, K3_NC, K3_NCW, K3_PPT, K3_ST, K3_NHE, false>
// pipelined block Jacobi (R-25): exact (lean cold tier: the z_hat / w_hat
// work would otherwise spill) and plain dots
#ifndef PBCG_PIPE_NH
#define PBCG_PIPE_NH 3
#endif
#define K2SX k2_stream<PBCG_PIPE_NH, K2_NC - 1, S_NCW, K2_PPT, K2_ST, K2_NHE, true, true>
#define K3SX k3_stream<PBCG_PIPE_NH, K3_NC - 1, S_NCW, K3_PPT, K3_ST, K3_NHE, true, true>  // 7 warps per group: 128 registers
#define K2SXP k2_stream<K2_NH, K2_NC, S_NCW, K2_PPT, K2_ST, K2_NHE, false, true>
#define K3SXP k3_stream<K3_NH, K3_NC, K3_NCW, K3_PPT, K3_ST, K3_NHE, false, true>
#define XDS exdot_stream<X_NH, X_NL, X_NCW, XD_PPT, XD_ST>
#define XDS2 exdot_stream<X_NH, X_NL, X_NCW, XD_PPT, XD_ST, 2>
static constexpr size_t ring_bytes(int nv, int ncw, int ppt, int stages) {
    return sizeof(double) * (size_t)stages * nv * (2 * ncw * 32 * ppt) + 2 * sizeof(uint64_t) * stages;
}
static constexpr size_t K2_SMEM = ring_bytes(8, S_NCW, K2_PPT, K2_ST);
static constexpr size_t K3_SMEM = ring_bytes(7, K3_NCW, K3_PPT, K3_ST);
static constexpr size_t K3X_SMEM = ring_bytes(7, S_NCW, K3_PPT, K3_ST);  // the pipelined block Jacobi's K3
static constexpr size_t XD_SMEM = ring_bytes(2, X_NCW, XD_PPT, XD_ST);
static constexpr int STREAM_THREADS = (X_NCW + 1) * 32;      // exdot: 1 dot group
static constexpr int KSTREAM_THREADS = (2 * S_NCW + 1) * 32;  // K2: 2 dot groups
static constexpr int K3_THREADS = (2 * K3_NCW + 1) * 32;       // K3: 2 dot groups
static constexpr size_t K2L_SMEM = ring_bytes(8, K2L_NCW, K2_PPT, K2_ST), K3L_SMEM = ring_bytes(7, K3L_NCW, K3_PPT, K3_ST);
static constexpr int K2L_THREADS = (2 * K2L_NCW + 1) * 32, K3L_THREADS = (2 * K3L_NCW + 1) * 32;


static int stream_attrs() {
    static int done = 0;
    if (done) return PBCG_OK;
    CUDA_TRY(cudaFuncSetAttribute((const void *)K2S, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K3S, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K2SP, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K2SL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2L_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K3SL, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3L_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K3SP, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K2SX, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K3SX, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3X_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K2SXP, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K2_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)K3SXP, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)XDS, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XD_SMEM));
    CUDA_TRY(cudaFuncSetAttribute((const void *)XDS2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)XD_SMEM));
    done = 1;
    return PBCG_OK;
}

static int stream_grid(pbcg_handle *h, int64_t n, int rows_per_tile) {
    const int64_t tiles = (n + rows_per_tile - 1) / rows_per_tile;
    return (int)std::max<int64_t>(1, std::min<int64_t>(h ? h->nsm : 148, tiles));
}

static int launch_xd1(pbcg_handle *h, const MultiDotArgs &a) {
    RC_TRY(stream_attrs());
    XDS<<<stream_grid(h, a.n, TileGeo<X_NCW, XD_PPT>::T), STREAM_THREADS, XD_SMEM, h->stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    return PBCG_OK;
}

static int launch_xd2(pbcg_handle *h, const MultiDotArgs &a) {  // (x,y), (y,y)
    RC_TRY(stream_attrs());
    XDS2<<<stream_grid(h, a.n, TileGeo<X_NCW, XD_PPT>::T), STREAM_THREADS, XD_SMEM, h->stream>>>(a);
    CUDA_TRY(cudaGetLastError());
    return PBCG_OK;
}

static int launch_k2(pbcg_handle *h, Rank &R, int fin, cudaStream_t st) {
    // fin = 1: the last CTA rounds and runs the scalar step; fin = 0: publish only (finalize_kernel follows)
    K2Args a{R.n, R.r, R.rh, R.w(), R.t, R.v, R.p, R.s, R.z(), R.q, R.y, R.sc, R.gacc[1], fin ? R.tickets + 1 : nullptr, R.hist, fin, R.part[1],
             R.pipe ? R.bji : nullptr, R.pipe ? R.zhpad + R.own_off : nullptr, R.rb + R.n == R.ng};
    if (R.pipe) {
        if (h->dot_mode == PBCG_DOT_PLAIN)
            launch_ex(K2SXP, dim3(stream_grid(h, R.n, TileGeo<S_NCW, K2_PPT>::T)), dim3(KSTREAM_THREADS), K2_SMEM, st,
                      pdl_for(R), a);
        else
            launch_ex(K2SX, dim3(stream_grid(h, R.n, TileGeo<S_NCW, K2_PPT>::T)), dim3(KSTREAM_THREADS), K2_SMEM, st,
                      pdl_for(R), a);
    } else if (h->dot_mode == PBCG_DOT_PLAIN) {
        launch_ex(K2SP, dim3(stream_grid(h, R.n, TileGeo<S_NCW, K2_PPT>::T)), dim3(KSTREAM_THREADS), K2_SMEM, st,
                  pdl_for(R), a);
    } else if (R.n < LEAN_ROWS) {
        launch_ex(K2SL, dim3(stream_grid(h, R.n, TileGeo<K2L_NCW, K2_PPT>::T)), dim3(K2L_THREADS), K2L_SMEM, st,
                  pdl_for(R), a);
    } else {
        launch_ex(K2S, dim3(stream_grid(h, R.n, TileGeo<S_NCW, K2_PPT>::T)), dim3(KSTREAM_THREADS), K2_SMEM, st,
                  pdl_for(R), a);
    }
    CUDA_TRY(cudaGetLastError());
    return PBCG_OK;
}

static int launch_k3(pbcg_handle *h, Rank &R, int fin, cudaStream_t st) {
    K3Args a{R.n, R.rh, R.p, R.q, R.y, R.t, R.v, R.x, R.r, R.w(), R.sc, R.gacc[2], fin ? R.tickets + 2 : nullptr, R.hist, fin, R.part[2],
             R.pipe ? R.bji : nullptr, R.pipe ? R.whpad + R.own_off : nullptr, R.rb + R.n == R.ng};
    if (R.pipe) {
        if (h->dot_mode == PBCG_DOT_PLAIN)
            launch_ex(K3SXP, dim3(stream_grid(h, R.n, TileGeo<K3_NCW, K3_PPT>::T)), dim3(K3_THREADS), K3_SMEM, st,
                      pdl_for(R), a);
        else
            launch_ex(K3SX, dim3(stream_grid(h, R.n, TileGeo<S_NCW, K3_PPT>::T)), dim3(KSTREAM_THREADS), K3X_SMEM, st,
                      pdl_for(R), a);
    } else if (h->dot_mode == PBCG_DOT_PLAIN) {
        launch_ex(K3SP, dim3(stream_grid(h, R.n, TileGeo<K3_NCW, K3_PPT>::T)), dim3(K3_THREADS), K3_SMEM, st,
                  pdl_for(R), a);
    } else if (R.n < LEAN_ROWS) {
        launch_ex(K3SL, dim3(stream_grid(h, R.n, TileGeo<K3L_NCW, K3_PPT>::T)), dim3(K3L_THREADS), K3L_SMEM, st,
                  pdl_for(R), a);
    } else {
        launch_ex(K3S, dim3(stream_grid(h, R.n, TileGeo<K3_NCW, K3_PPT>::T)), dim3(K3_THREADS), K3_SMEM, st,
                  pdl_for(R), a);
    }
    CUDA_TRY(cudaGetLastError());
    return PBCG_OK;
}

static int enqueue_alg1(pbcg_handle *h);

static int enqueue_iteration(pbcg_handle *h) {
    if (h->method == PBCG_METHOD_BICGSTAB) return enqueue_alg1(h);
    cudaStream_t st = h->stream;
    if (!multi(h)) {
        // single rank: the rounding + scalar step of each phase (finalize_kernel,
        // 1 CTA) runs on the side stream while the SpMV that does not need
        // its scalars runs on the main stream -- the same fork/join as the
        // multi-rank allreduce, minus the communication.
        Rank &R = h->R[0];
        RC_TRY(launch_k2(h, R, 0, st));
        CUDA_TRY(cudaEventRecord(h->ev[4], st));
        CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev[4], 0));
        if (h->dot_mode == PBCG_DOT_PLAIN) RC_TRY(reduce_finalize<4>(h, 1, PH_A, h->side, nullptr, nullptr));
        else finalize_kernel<4><<<1, 128, 0, h->side>>>(R.gacc[1], PH_A, R.sc, R.hist, nullptr, nullptr);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaEventRecord(h->ev[5], h->side));
        RC_TRY(launch_spmv(h, R, SPMV_PLAIN, padbuf(R, 0), R.v, nullptr, nullptr, true, st));
        CUDA_TRY(cudaStreamWaitEvent(st, h->ev[5], 0));
        RC_TRY(launch_k3(h, R, 0, st));
        CUDA_TRY(cudaEventRecord(h->ev[6], st));
        CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev[6], 0));
        if (h->dot_mode == PBCG_DOT_PLAIN) RC_TRY(reduce_finalize<3>(h, 2, PH_B, h->side, nullptr, nullptr));
        else finalize_kernel<3><<<1, 128, 0, h->side>>>(R.gacc[2], PH_B, R.sc, R.hist, nullptr, nullptr);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaEventRecord(h->ev[7], h->side));
        RC_TRY(launch_spmv(h, R, SPMV_PLAIN, padbuf(R, 1), R.t, nullptr, nullptr, true, st));
        CUDA_TRY(cudaStreamWaitEvent(st, h->ev[7], 0));
        return PBCG_OK;
    }
    // halo + SpMV of padded buffer `which` into y: with a split, the interior
    // rows run while the halo exchange runs on cstream (joined before the
    // boundary rows; "communication hiding" applied to the halo too)
    const int reserve = (h->comm && h->nranks > 1) ? SPMV_COMM_SMS : 0;
    auto halo_spmv = [&](int which, double *Rank::*ymem, int evi) -> int {
        bool split = false;
        for (auto &R : h->R) split |= R.split;
        if (!split) {
            RC_TRY(halo(h, which));
            for (auto &R : h->R) {
                double *xp = padbuf(R, which);
                RC_TRY(launch_spmv(h, R, SPMV_PLAIN, xp, R.*ymem, nullptr, nullptr, true, st));
            }
            return PBCG_OK;
        }
        CUDA_TRY(cudaEventRecord(h->evh[evi], st));  // the vector to exchange is complete
        CUDA_TRY(cudaStreamWaitEvent(h->cstream, h->evh[evi], 0));
        RC_TRY(halo(h, which, h->cstream));
        CUDA_TRY(cudaEventRecord(h->evh[evi + 1], h->cstream));
        for (auto &R : h->R) {
            double *xp = padbuf(R, which);
            RC_TRY(launch_spmv(h, R, SPMV_PLAIN, xp, R.*ymem, nullptr, nullptr, true, st, SP_INTERIOR, reserve));
        }
        CUDA_TRY(cudaStreamWaitEvent(st, h->evh[evi + 1], 0));
        for (auto &R : h->R) {
            double *xp = padbuf(R, which);
            RC_TRY(launch_spmv(h, R, SPMV_PLAIN, xp, R.*ymem, nullptr, nullptr, true, st, SP_BOUNDARY));
        }
        return PBCG_OK;
    };
    if (h->V > 1) {  // virtual ranks: same dataflow, the reductions serialised on the main stream
        for (auto &R : h->R) RC_TRY(launch_k2(h, R, 0, st));
        RC_TRY(reduce_finalize<4>(h, 1, PH_A, st, nullptr, nullptr));
        RC_TRY(halo_spmv(0, &Rank::v, 0));
        for (auto &R : h->R) RC_TRY(launch_k3(h, R, 0, st));
        RC_TRY(reduce_finalize<3>(h, 2, PH_B, st, nullptr, nullptr));
        RC_TRY(halo_spmv(1, &Rank::t, 2));
        return PBCG_OK;
    }
    // real ranks: phase allreduce on the side stream overlaps halo + SpMV (l.90)
    Rank &R = h->R[0];
    RC_TRY(launch_k2(h, R, 0, st));
    CUDA_TRY(cudaEventRecord(h->ev[0], st));
    CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev[0], 0));
    RC_TRY(reduce_finalize<4>(h, 1, PH_A, h->side, nullptr, nullptr));
    CUDA_TRY(cudaEventRecord(h->ev[1], h->side));
    RC_TRY(halo_spmv(0, &Rank::v, 0));
    CUDA_TRY(cudaStreamWaitEvent(st, h->ev[1], 0));
    RC_TRY(launch_k3(h, R, 0, st));
    CUDA_TRY(cudaEventRecord(h->ev[2], st));
    CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev[2], 0));
    RC_TRY(reduce_finalize<3>(h, 2, PH_B, h->side, nullptr, nullptr));
    CUDA_TRY(cudaEventRecord(h->ev[3], h->side));
    RC_TRY(halo_spmv(1, &Rank::t, 2));
    CUDA_TRY(cudaStreamWaitEvent(st, h->ev[3], 0));
    return PBCG_OK;
}

// ----------------------------------------------------------------------------
// setup / destroy
// ----------------------------------------------------------------------------
// Packed SELL-P chunks (spmv_sellp_kernel): explicit-slot counts on the
// device, chunk byte offsets on the host (prefix sum), then the scatter.
static int build_sellp(pbcg_handle *h, Rank &R) {
    using Geo = SellPGeo<PS_SPS>;
    const int32_t *rec = R.use_slots ? R.slot_rec : nullptr;
    const int g = (int)std::min<int64_t>((R.nslices + 255) / 256, 65535);
    sellp_count_kernel<<<g, 256, 0, h->stream>>>(R.nslices, R.slice_off, rec, R.nexp);
    CUDA_TRY(cudaGetLastError());
    std::vector<uint8_t> ne(R.nslices);
    CUDA_TRY(cudaMemcpyAsync(ne.data(), R.nexp, R.nslices, cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    std::vector<int64_t> off(R.nchunks + 1, 0);
    for (int64_t c = 0; c < R.nchunks; ++c) {
        const int64_t s0 = c * PS_SPS, s1 = std::min<int64_t>(s0 + PS_SPS, R.nslices);
        int64_t nx = 0;
        for (int64_t s = s0; s < s1; ++s) nx += 32 * ne[s];
        const int64_t nv = R.h_slice_off[s1] - R.h_slice_off[s0];
        off[c + 1] = off[c] + ((Geo::H + 8 * nv + 4 * nx + 15) & ~int64_t(15));
    }
    if (off[R.nchunks] > R.blob_cap) return fail(PBCG_ENOMEM, "sellp: packed chunks exceed their bound");
    R.blob_bytes = off[R.nchunks];
    int64_t mx = 0;
    for (int64_t c = 0; c < R.nchunks; ++c) mx = std::max(mx, off[c + 1] - off[c]);
    R.ps_stage = (int)((mx + 127) & ~int64_t(127));
    R.ps_stages = (int)std::min<int64_t>(PS_MAXSTAGES, (PS_SMEM_MAX - 256) / R.ps_stage);
    if (R.ps_stages < 2) {  // chunks too large for a double-buffered ring: register-pipelined kernel
        R.spmv_kind = SPMV_K_PIPE;
        return PBCG_OK;
    }
    CUDA_TRY(cudaMemcpyAsync(R.blob_off, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, h->stream));
    CUDA_TRY(cudaMemsetAsync(R.blob, 0, (size_t)R.blob_bytes, h->stream));
    SellMat M = R.mat();
    M.slot_rec = rec;
    const int gf = (int)std::min<int64_t>((R.nslices + 7) / 8, 65535);
    sellp_fill_kernel<PS_SPS><<<gf, 256, 0, h->stream>>>(R.n, R.nslices, M, R.nexp, R.blob_off, R.blob);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(h->stream));  // off (host vector) must outlive the copy
    return PBCG_OK;
}

// SELL-V chunks (spmv_sellv_kernel): nonzeros per slice on the device, the
// byte-bounded chunking on the host (at most PV_NCW slices and PV_CAP bytes
// per chunk, or one slice), then the scatter.
static int build_sellv(pbcg_handle *h, Rank &R) {
    const int64_t ns = R.nslices;
    int32_t *d_tmp = nullptr;  // [nnz per slice | cs | vs | x lo per slice | x hi per slice]
    CUDA_TRY(cudaMalloc(&d_tmp, sizeof(int32_t) * (5 * ns + 2)));
    int32_t *d_cnt = d_tmp, *d_cs = d_tmp + ns, *d_vs = d_tmp + 2 * ns + 1, *d_lo = d_tmp + 3 * ns + 2,
            *d_hi = d_tmp + 4 * ns + 2;
    std::vector<int32_t> cnt(ns), slo(ns), shi(ns);
    {
        const int g = (int)std::min<int64_t>((ns + 255) / 256, 65535);
        sellv_count_kernel<<<g, 256, 0, h->stream>>>(R.n, ns, R.row_len, d_cnt);
        const int gx = (int)std::min<int64_t>((ns + 7) / 8, 65535);
        sellv_xrange_kernel<<<gx, 256, 0, h->stream>>>(R.n, ns, R.mat(), d_lo, d_hi);
        cudaError_t ce = cudaGetLastError();
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(cnt.data(), d_cnt, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, h->stream);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(slo.data(), d_lo, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, h->stream);
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(shi.data(), d_hi, sizeof(int32_t) * ns, cudaMemcpyDeviceToHost, h->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);
        if (ce != cudaSuccess) {
            cudaFree(d_tmp);
            return fail(PBCG_ECUDA, "sellv: %s", cudaGetErrorString(ce));
        }
    }
    auto bytes = [](int64_t nsl, int64_t nv) { return (sellv_hdr_bytes((int)nsl) + 12 * nv + 15) & ~int64_t(15); };
    std::vector<int32_t> cs, vs(ns), clo, chi;
    std::vector<int64_t> off;
    // chunks of consecutive slices: at most `ncw` slices and `cap` bytes (or one
    // slice); then each chunk's x range and the ring geometry: the most stages
    // (>= min_st) whose x window fits next to `stage` bytes per stage
    auto plan = [&](int64_t cap, int ncw, bool gld, int min_st) {
        cs.assign(1, 0);
        off.assign(1, 0);
        int64_t mx = 0;
        for (int64_t s0 = 0; s0 < ns;) {
            int64_t s1 = s0, nv = 0;
            while (s1 < ns && (s1 == s0 || (s1 - s0 < ncw && bytes(s1 + 1 - s0, nv + cnt[s1]) <= cap))) {
                vs[s1] = (int32_t)nv;
                nv += cnt[s1++];
            }
            const int64_t b = bytes(s1 - s0, nv);
            mx = std::max(mx, b);
            off.push_back(off.back() + b);
            cs.push_back((int32_t)s1);
            s0 = s1;
        }
        const int64_t nch = (int64_t)cs.size() - 1;
        R.nchunks = nch;
        R.blob_bytes = off.back();
        R.ps_stage = gld ? (sellv_hdr_bytes(ncw) + 127) & ~127 : (int)((mx + 127) & ~int64_t(127));
        clo.assign(nch, INT32_MAX);
        chi.assign(nch, -1);
        std::vector<int64_t> H(nch);  // running maximum of the chunks' even-rounded upper x index
        for (int64_t c = 0; c < nch; ++c) {
            for (int64_t q = cs[c]; q < cs[c + 1]; ++q) {
                clo[c] = std::min(clo[c], slo[q]);
                chi[c] = std::max(chi[c], shi[q]);
            }
            H[c] = std::max<int64_t>(c ? H[c - 1] : 0, (chi[c] + 1) & ~1);
        }
        R.ps_stages = 0;
        R.ps_xr = 0;
        R.pv_gld = gld;
        for (int S = PV_MAXSTAGES; S >= min_st && !R.ps_stages; --S) {
            int64_t span = 0;
            for (int64_t c = 0; c < nch; ++c)
                if (clo[c] != INT32_MAX) span = std::max<int64_t>(span, H[std::min<int64_t>(c + S - 1, nch - 1)] - clo[c]);
            // any multiple of 64 doubles (the consumers reduce i mod XR with one
            // compare per gather): C4's +-5000 band needs ~85 KB instead of the
            // 128 KB of a power of two, which leaves room for 6 ring stages
            const int64_t xr = std::max<int64_t>(1024, (span + 4 + 63) & ~int64_t(63));
            // the matrix through the ring (gld = false) only for narrow windows:
            // C4's +-5000 band (85 KB) ran at 356 us that way with 6 stages,
            // against 299 us with the consumers loading the matrix (gld)
            if (!gld && 8 * xr > PV_TMA_MAX_WINDOW) continue;
            if ((int64_t)S * R.ps_stage + 8 * xr + 16 * S + 256 <= PS_SMEM_MAX) {
                R.ps_stages = S;
                R.ps_xr = (int)xr;
            }
        }
        return R.ps_stages > 0 && R.blob_bytes <= R.blob_cap - 2048;
    };
    // the matrix through the ring when the window leaves a deep one; else
    // the matrix loaded by the consumers, only chunk headers in the ring
    // (PBCG_SELLV_MODE=tma|gld forces one, for A/B runs)
    const char *em = getenv("PBCG_SELLV_MODE");
    bool ok = false;
    for (int64_t cap : {(int64_t)PV_CAP, (int64_t)PV_CAP * 5 / 6, (int64_t)PV_CAP * 2 / 3})
        if (!ok && (!em || strcmp(em, "gld") != 0)) ok = plan(cap, PV_NCW, false, PV_MIN_WIN_STAGES);
    if (!ok && (!em || strcmp(em, "tma") != 0)) ok = plan(INT64_MAX / 4, PV_NCW_G, true, 2);
    if (!ok) {  // x window wider than shared memory (not banded): one row per thread
        cudaFree(d_tmp);
        R.spmv_kind = SPMV_K_PLAIN;
        return PBCG_OK;
    }
    R.h_cs = cs;
    const int64_t nch = R.nchunks;
    cudaError_t ce = cudaMemcpyAsync(R.blob_off, off.data(), sizeof(int64_t) * off.size(), cudaMemcpyHostToDevice, h->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(R.cxlo, clo.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice, h->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(R.cxhi, chi.data(), sizeof(int32_t) * nch, cudaMemcpyHostToDevice, h->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(d_cs, cs.data(), sizeof(int32_t) * cs.size(), cudaMemcpyHostToDevice, h->stream);
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(d_vs, vs.data(), sizeof(int32_t) * ns, cudaMemcpyHostToDevice, h->stream);
    if (ce == cudaSuccess) ce = cudaMemsetAsync(R.blob, 0, (size_t)R.blob_bytes + 2048, h->stream);
    if (ce == cudaSuccess) {
        const int gf = (int)std::min<int64_t>((ns + 7) / 8, 65535);
        sellv_fill_kernel<<<gf, 256, 0, h->stream>>>(R.n, ns, R.mat(), d_cs, d_vs, R.nchunks, R.blob_off, R.blob);
        ce = cudaGetLastError();
    }
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);  // host vectors must outlive the copies
    cudaFree(d_tmp);
    if (ce != cudaSuccess) return fail(PBCG_ECUDA, "sellv: %s", cudaGetErrorString(ce));
    return PBCG_OK;
}

static int copy_own_to_pad(pbcg_handle *h, double *Rank::*src_member, int which);
static int small_grid_for(pbcg_handle *h);

// Right Jacobi (NEXT-3, R-22): d = diag(A) per rank, d into the padded
// x layout + halo (the columns' diagonals), then A' = A D^-1 in the SELL.
// 2x2 block Jacobi (R-23) after the SELL of B's pattern is built: M and M^-1
// of every own block, the columns of M^-1 in the padded x layout (z / w
// buffers, halo exchanged like a vector), then B = A M^-1 in place.
static int bj_setup(pbcg_handle *h, const pbcg_csr_local *A0) {
    for (auto &R : h->R) {
        if (R.rb & 1) return fail(PBCG_EINVAL, "block jacobi: every rank's first row must be even (whole 2x2 blocks)");
        if (R.n == 0) continue;
        const int32_t *rp = A0->row_ptr + (h->V > 1 ? R.rb : 0);
        const int g = (int)std::min<int64_t>((R.n + 511) / 512, 65535);
        bj_blocks_kernel<<<g, 256, 0, h->stream>>>(R.n, R.rb, h->n_global, rp, A0->col_idx, A0->values, R.bjm,
                                                   R.bji, R.zpad + R.own_off, R.wpad + R.own_off, R.bad);
        CUDA_TRY(cudaGetLastError());
    }
    RC_TRY(halo(h, 0));
    RC_TRY(halo(h, 1));
    for (auto &R : h->R) {
        if (R.n == 0) continue;
        const int g = (int)std::min<int64_t>((R.n + 255) / 256, 65535);
        bj_values_kernel<<<g, 256, 0, h->stream>>>(R.n, h->n_global, R.buf_lo, R.slice_off, R.row_len, R.sval,
                                                   R.scol, R.zpad, R.wpad);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (auto &R : h->R) {
        int bad = 0;
        CUDA_TRY(cudaMemcpy(&bad, R.bad, sizeof(int), cudaMemcpyDeviceToHost));
        if (bad & 4) return fail(PBCG_EINVAL, "block jacobi: singular or non-finite 2x2 diagonal block");
        CUDA_TRY(cudaMemset(R.zpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo)));
        CUDA_TRY(cudaMemset(R.wpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo)));
    }
    return PBCG_OK;
}

// Pipelined 2x2 block Jacobi (R-25): M and M^-1 of every own block; the
// matrix stays A (the iteration applies M^-1 to z and w in K2 / K3).
static int bj_pipe_setup(pbcg_handle *h, const pbcg_csr_local *A0) {
    for (auto &R : h->R) {
        if (R.rb & 1) return fail(PBCG_EINVAL, "block jacobi: every rank's first row must be even (whole 2x2 blocks)");
        R.pipe = true;
        R.ng = h->n_global;
        CUDA_TRY(cudaMemsetAsync(R.zhpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo), h->stream));
        CUDA_TRY(cudaMemsetAsync(R.whpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo), h->stream));
        if (R.n == 0) continue;
        const int32_t *rp = A0->row_ptr + (h->V > 1 ? R.rb : 0);
        const int g = (int)std::min<int64_t>((R.n + 511) / 512, 65535);
        // the M^-1 column outputs (stored-B mode) land in the unused own part of xpad
        bj_blocks_kernel<<<g, 256, 0, h->stream>>>(R.n, R.rb, h->n_global, rp, A0->col_idx, A0->values, R.bjm,
                                                   R.bji, R.xpad + R.own_off, R.tmp, R.bad);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (auto &R : h->R) {
        int bad = 0;
        CUDA_TRY(cudaMemcpy(&bad, R.bad, sizeof(int), cudaMemcpyDeviceToHost));
        if (bad & 4) return fail(PBCG_EINVAL, "block jacobi: singular or non-finite 2x2 diagonal block");
        CUDA_TRY(cudaMemset(R.xpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo)));
    }
    return PBCG_OK;
}

static int jacobi_scale(pbcg_handle *h, const pbcg_csr_local *A) {
    for (auto &R : h->R) {
        if (R.n == 0) continue;
        const int32_t *rp = A->row_ptr + (h->V > 1 ? R.rb : 0);
        const int g = (int)std::min<int64_t>((R.n + 255) / 256, 65535);
        diag_kernel<<<g, 256, 0, h->stream>>>(R.n, R.rb, rp, A->col_idx, A->values, R.dg, R.bad);
        CUDA_TRY(cudaGetLastError());
    }
    RC_TRY(copy_own_to_pad(h, &Rank::dg, 2));
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) {
        if (R.n == 0) continue;
        const int g = (int)std::min<int64_t>((R.n + 255) / 256, 65535);
        sell_colscale_kernel<<<g, 256, 0, h->stream>>>(R.n, R.slice_off, R.row_len, R.sval, R.scol, R.xpad);
        CUDA_TRY(cudaGetLastError());
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    for (auto &R : h->R) {
        int bad = 0;
        CUDA_TRY(cudaMemcpy(&bad, R.bad, sizeof(int), cudaMemcpyDeviceToHost));
        if (bad & 4) return fail(PBCG_EINVAL, "jacobi: zero or missing diagonal entry");
    }
    return PBCG_OK;
}

// Multi-rank halo overlap: per rank, the longest run of slices that read no
// halo entry is the interior (for the SELL-P kernel: whole chunks inside it).
// PBCG_SPLIT=0 turns the overlap off.
static int plan_split(pbcg_handle *h) {
    const char *e = getenv("PBCG_SPLIT");
    if (e && e[0] == '0') return PBCG_OK;
    for (auto &R : h->R) {
        R.split = false;
        if (R.n == 0 || R.nslices < 4) continue;
        uint8_t *d_flag = nullptr;
        CUDA_TRY(cudaMalloc(&d_flag, (size_t)R.nslices));
        const int g = (int)std::min<int64_t>((R.nslices + 7) / 8, 65535);
        sell_halo_flags_kernel<<<g, 256, 0, h->stream>>>(R.n, R.nslices, R.slice_off, R.row_len, R.scol, R.own_off,
                                                         R.own_off + R.n, d_flag);
        std::vector<uint8_t> f(R.nslices);
        cudaError_t ce = cudaGetLastError();
        if (ce == cudaSuccess) ce = cudaMemcpyAsync(f.data(), d_flag, (size_t)R.nslices, cudaMemcpyDeviceToHost, h->stream);
        if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);
        cudaFree(d_flag);
        if (ce != cudaSuccess) return fail(PBCG_ECUDA, "plan_split: %s", cudaGetErrorString(ce));
        int64_t best0 = 0, best1 = 0;
        for (int64_t s0 = 0; s0 < R.nslices;) {  // longest run of interior slices
            if (f[s0]) { ++s0; continue; }
            int64_t s1 = s0;
            while (s1 < R.nslices && !f[s1]) ++s1;
            if (s1 - s0 > best1 - best0) { best0 = s0; best1 = s1; }
            s0 = s1;
        }
        int64_t lo = best0, hi = best1, units = R.nslices;
        if (R.spmv_kind == SPMV_K_TMA) {
            lo = (best0 + PS_SPS - 1) / PS_SPS;
            hi = best1 / PS_SPS;
            units = R.nchunks;
        } else if (R.spmv_kind == SPMV_K_TMAV) {  // whole chunks inside [best0, best1)
            lo = std::lower_bound(R.h_cs.begin(), R.h_cs.end(), (int32_t)best0) - R.h_cs.begin();
            hi = std::upper_bound(R.h_cs.begin(), R.h_cs.end(), (int32_t)best1) - R.h_cs.begin() - 1;
            units = R.nchunks;
        }
        if (hi - lo >= units / 4) {  // worth a second launch
            R.split = true;
            R.in_lo = lo;
            R.in_hi = hi;
        }
    }
    return PBCG_OK;
}

// Chunked start (pbicgstab_start with x0 = 0 and a host b): the copy of b
// streams in START_NCH chunks and the init work of each chunk -- the scans
// and copies, w0 = A r0 and t0 = A w0 over its rows, its share of the two
// init dots -- runs as soon as the chunks it reads have landed (a pipeline
// lagging one and two chunks).  Planned here: chunk boundaries on SpMV unit
// boundaries that are also 256-row window boundaries (so a chunk's
// positions are its rows), and the largest row each chunk's rows read,
// which must lie in the next chunk at most.  One rank, SELL-P or the slice
// kernels; otherwise start copies b whole.
static constexpr int START_NCH = 16;
static int plan_start(pbcg_handle *h) {
    if (h->R.size() != 1 || h->comm) return PBCG_OK;
    Rank &R = h->R[0];
    R.st_row.clear();
    R.st_u.clear();
    if (R.n < (1 << 20) || R.pipe || R.spmv_kind == SPMV_K_TMAV) return PBCG_OK;
    int64_t *d_x = nullptr;
    CUDA_TRY(cudaMalloc(&d_x, sizeof(int64_t) * (size_t)R.nslices));
    const int g = (int)std::min<int64_t>((R.nslices + 7) / 8, 65535);
    sell_xmax_kernel<<<g, 256, 0, h->stream>>>(R.n, R.nslices, R.slice_off, R.row_len, R.scol, d_x);
    std::vector<int64_t> xm(R.nslices);
    cudaError_t ce = cudaGetLastError();
    if (ce == cudaSuccess) ce = cudaMemcpyAsync(xm.data(), d_x, sizeof(int64_t) * R.nslices, cudaMemcpyDeviceToHost, h->stream);
    if (ce == cudaSuccess) ce = cudaStreamSynchronize(h->stream);
    cudaFree(d_x);
    if (ce != cudaSuccess) return fail(PBCG_ECUDA, "plan_start: %s", cudaGetErrorString(ce));
    const bool tma = R.spmv_kind == SPMV_K_TMA;
    const int64_t su = tma ? PS_SPS : 1;                 // slices per unit
    const int64_t ustep = tma ? 4 : 8;                  // units per 256-row-aligned step (3,840 / 256 rows)
    const int64_t units = tma ? R.nchunks : R.nslices;
    std::vector<int64_t> ub(START_NCH + 1), rb(START_NCH + 1);
    for (int k = 0; k <= START_NCH; ++k) {
        int64_t u = (units * k / START_NCH) / ustep * ustep;
        if (k == START_NCH) u = units;
        ub[k] = u;
        rb[k] = std::min<int64_t>(R.n, u * su * 32);
    }
    for (int k = 0; k < START_NCH; ++k) {
        if (rb[k + 1] <= rb[k]) return PBCG_OK;  // too few units for the chunks
        int64_t mx = -1;
        for (int64_t sl = ub[k] * su; sl < std::min<int64_t>(ub[k + 1] * su, R.nslices); ++sl) mx = std::max(mx, xm[sl]);
        const int64_t row = mx - R.own_off;  // x-buffer index -> row (one rank: no halo)
        if (k + 2 <= START_NCH && row >= rb[k + 2]) return PBCG_OK;  // reads beyond the next chunk
    }
    R.st_row = rb;
    R.st_u = ub;
    return PBCG_OK;
}

extern "C" int pbicgstab_setup(const pbcg_csr_local *A, const pbcg_dist *d, void *stream, void *workspace,
                               size_t workspace_bytes, pbcg_handle **out) {
    NvtxRange nvtx_("pbcg.setup");
    if (!out) return fail(PBCG_EINVAL, "out == NULL");
    *out = nullptr;
    auto *h = new pbcg_handle();
    std::unique_ptr<pbcg_handle> guard(h);
    h->stream = (cudaStream_t)stream;
    CUDA_TRY(cudaGetDevice(&h->dev));
    CUDA_TRY(cudaDeviceGetAttribute(&h->nsm, cudaDevAttrMultiProcessorCount, h->dev));
    const int nranks = d ? std::max(1, d->nranks) : 1;
    // 2x2 block Jacobi: the layout is B's (pattern expanded to whole column
    // blocks); A0 keeps the caller's matrix for the blocks of M
    const pbcg_csr_local *A0 = A;
    BjCsr bj;
    if (A && d && d->precond == PBCG_PRECOND_BJACOBI2) {
        RC_TRY(validate_csr(A, d));
        RC_TRY(bj_expand(A, bj));
        A = &bj.B;
    }
    // communicators first: real ranks need the allgathered row ranges + hulls
    std::vector<int64_t> all_ranges;
    std::vector<int32_t> h_rp;
    const bool force_comm = d && d->comm_mode == 1 && nranks == 1 && d->virtual_ranks <= 1;
    if (nranks > 1 || force_comm) {
        if (!nccl_available()) return fail(PBCG_ENCCL, "nranks > 1 but libnccl.so.2 could not be loaded");
        ncclUniqueId uid;
        if (d->nccl_uid) memcpy(&uid, d->nccl_uid, sizeof(uid));
        else if (force_comm) NCCL_TRY(g_nccl.GetUniqueId(&uid));
        else return fail(PBCG_EINVAL, "nranks > 1 needs nccl_uid");
        h->comm = true;
        // two communicators (halo on the main stream, reductions on the side
        // stream, so they can run concurrently); one unique id bootstraps one
        // communicator, the second is split from it.  Each may use at most
        // NCCL_CTAS CTAs: the interior SpMV they overlap leaves SPMV_COMM_SMS
        // SMs free
        ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
        cfg.blocking = 1;
        cfg.minCTAs = 1;
        cfg.maxCTAs = nccl_ctas();
        cfg.commName = "pbcg_halo";
        ncclConfig_t cfg2 = cfg;
        cfg2.commName = "pbcg_reduce";
        if (g_nccl.CommInitRankConfig)
            NCCL_TRY(g_nccl.CommInitRankConfig(&h->comm_halo, nranks, uid, d->rank, &cfg));
        else
            NCCL_TRY(g_nccl.CommInitRank(&h->comm_halo, nranks, uid, d->rank));
        NCCL_TRY(g_nccl.CommSplit(h->comm_halo, 0, d->rank, &h->comm_red, &cfg2));
        // hull of my rows and the config hash, then allgather every rank's record
        RC_TRY(validate_csr(A, d));
        if (A && d->virtual_ranks > 1) return fail(PBCG_EINVAL, "virtual ranks need nranks == 1");
        int64_t mine[PBCG_RANK_REC] = {A ? A->row_begin : 0, A ? A->row_end : 0, 0, -1, 0};
        uint64_t hsh = 0;
        RC_TRY(pbcg_config_hash(A, d, &hsh));
        mine[4] = (int64_t)hsh;
        if (A) {
            std::vector<int64_t> b1 = {0, A->row_end - A->row_begin};
            std::vector<long long> hull;
            RC_TRY(compute_hulls(A, 1, b1, hull));
            if (hull[1] >= hull[0]) { mine[2] = hull[0]; mine[3] = hull[1]; }
        }
        int64_t *dbuf = nullptr;
        CUDA_TRY(cudaMalloc(&dbuf, sizeof(int64_t) * PBCG_RANK_REC * (nranks + 1)));
        CUDA_TRY(cudaMemcpy(dbuf, mine, sizeof(mine), cudaMemcpyHostToDevice));
        NCCL_TRY(g_nccl.AllGather(dbuf, dbuf + PBCG_RANK_REC, PBCG_RANK_REC, ncclInt64, h->comm_red, h->stream));
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        std::vector<int64_t> rec((size_t)PBCG_RANK_REC * nranks);
        CUDA_TRY(cudaMemcpy(rec.data(), dbuf + PBCG_RANK_REC, sizeof(int64_t) * rec.size(), cudaMemcpyDeviceToHost));
        cudaFree(dbuf);
        RC_TRY(pbcg_check_ranks(nranks, rec.data(), A ? A->n_global : 0, A ? 1 : 0));
        all_ranges.resize(4 * (size_t)nranks);
        for (int k = 0; k < nranks; ++k)
            for (int j = 0; j < 4; ++j) all_ranges[4 * k + j] = rec[(size_t)PBCG_RANK_REC * k + j];
    }
    RC_TRY(prepare(h, A, d, h_rp, h->comm ? &all_ranges : nullptr));
    h->nranks = nranks;
    h->rank = d ? d->rank : 0;
    const size_t need = total_size(h);
    h->ws_need = need;
    if (!workspace || workspace_bytes < need)
        return fail(PBCG_ENOMEM, "workspace too small: need %zu bytes, got %zu", need, workspace_bytes);
    Carver C{(char *)(((uintptr_t)workspace + 255) & ~uintptr_t(255))};
    for (auto &R : h->R) carve_rank(C, R, h->hist_cap, h->comm_only, h->precond);
    carve_handle_extra(C, h);
    // zero reduction state
    for (auto &R : h->R) {
        for (int k = 0; k < NPH; ++k) CUDA_TRY(cudaMemsetAsync(R.gacc[k], 0, sizeof(long long) * GW4, h->stream));
        for (int k = 0; k < NPH; ++k) CUDA_TRY(cudaMemsetAsync(R.part[k], 0, sizeof(double) * PLAIN_GRID * 4, h->stream));
        CUDA_TRY(cudaMemsetAsync(R.tickets, 0, sizeof(unsigned) * 16, h->stream));
        CUDA_TRY(cudaMemsetAsync(R.sc, 0, sizeof(Scalars), h->stream));
        CUDA_TRY(cudaMemsetAsync(R.bad, 0, sizeof(int) * 4, h->stream));
    }
    {
        std::vector<long long *> vg((size_t)NPH * h->V);
        for (int ph = 0; ph < NPH; ++ph)
            for (int v = 0; v < h->V; ++v) vg[(size_t)ph * h->V + v] = h->R[v].gacc[ph];
        CUDA_TRY(cudaMemcpyAsync(h->vgacc, vg.data(), sizeof(long long *) * vg.size(), cudaMemcpyHostToDevice, h->stream));
        std::vector<double *> vp((size_t)NPH * h->V);
        for (int ph = 0; ph < NPH; ++ph)
            for (int v = 0; v < h->V; ++v) vp[(size_t)ph * h->V + v] = h->R[v].part[ph];
        CUDA_TRY(cudaMemcpyAsync(h->vpart, vp.data(), sizeof(double *) * vp.size(), cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(cudaStreamSynchronize(h->stream));
    }
    if (!h->comm_only) {
        for (size_t v = 0; v < h->R.size(); ++v) {
            Rank &R = h->R[v];
            CUDA_TRY(cudaMemsetAsync(R.slice_off, 0, sizeof(int64_t) * (R.nslices + 16), h->stream));
            CUDA_TRY(cudaMemcpyAsync(R.slice_off, R.h_slice_off.data(), sizeof(int64_t) * (R.nslices + 1),
                                     cudaMemcpyHostToDevice, h->stream));
            CUDA_TRY(cudaMemsetAsync(R.row_len, 0, sizeof(int32_t) * R.nslices * 32, h->stream));
            if (!R.h_perm.empty())
                CUDA_TRY(cudaMemcpyAsync(R.perm, R.h_perm.data(), sizeof(int32_t) * R.h_perm.size(),
                                         cudaMemcpyHostToDevice, h->stream));
            CUDA_TRY(cudaMemsetAsync(R.zpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo), h->stream));
            CUDA_TRY(cudaMemsetAsync(R.wpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo), h->stream));
            CUDA_TRY(cudaMemsetAsync(R.xpad, 0, sizeof(double) * (R.buf_hi - R.buf_lo), h->stream));
            if (R.n > 0) {
                const int32_t *rp = A->row_ptr + (h->V > 1 ? R.rb : 0);
                const int grid = (int)std::min<int64_t>((R.n + 255) / 256, 65535);
                csr_to_sell_kernel<<<grid, 256, 0, h->stream>>>(R.n, rp, A->col_idx, A->values, A->n_global, R.buf_lo,
                                                                R.slice_off, R.row_len, R.sval, R.scol,
                                                                R.h_perm.empty() ? nullptr : R.perm, R.bad);
                CUDA_TRY(cudaGetLastError());
                // column offsets per slice-slot (index compression of the SELL)
                CUDA_TRY(cudaMemsetAsync(R.bad + 2, 0, sizeof(unsigned long long), h->stream));
                const int gs = (int)std::min<int64_t>((R.nslices + 7) / 8, 65535);
                sell_slot_records_kernel<<<gs, 256, 0, h->stream>>>(R.n, R.nslices, R.slice_off, R.row_len, R.scol,
                                                                     R.slot_rec,
                                                                     (unsigned long long *)(R.bad + 2));
                CUDA_TRY(cudaGetLastError());
            }
        }
        CUDA_TRY(cudaStreamSynchronize(h->stream));
        if (h->precond == PBCG_PRECOND_JACOBI) RC_TRY(jacobi_scale(h, A));
        if (h->precond == PBCG_PRECOND_BJACOBI2) RC_TRY(bj_setup(h, A0));
        if (h->precond == PBCG_PRECOND_BJACOBI2_PIPE) RC_TRY(bj_pipe_setup(h, A0));
        const char *es = getenv("PBCG_SELL_SLOTS");
        for (auto &R : h->R) {
            R.spmv_kind = spmv_kind_for(R, h->nsm);
            unsigned long long ne = 0;
            if (R.n > 0) CUDA_TRY(cudaMemcpy(&ne, R.bad + 2, sizeof(ne), cudaMemcpyDeviceToHost));
            // the slot records replace column ids in the packed SELL-P chunks
            // when they spare at least a quarter of them
            R.use_slots = R.spmv_kind == SPMV_K_TMA && !(es && es[0] == '0') && 4 * (int64_t)ne <= 3 * R.nnz;
            R.n_explicit = R.use_slots ? (int64_t)ne : R.nnz;
            int bad = 0;
            CUDA_TRY(cudaMemcpy(&bad, R.bad, sizeof(int), cudaMemcpyDeviceToHost));
            if (bad & 1) return fail(PBCG_EINVAL, "csr: column ids not strictly increasing / out of range");
            if (bad & 2) return fail(PBCG_ENONFINITE, "csr: NaN/Inf value");
            if (R.spmv_kind == SPMV_K_TMA) {
                if (R.blob && R.n > 0) RC_TRY(build_sellp(h, R));
                else R.spmv_kind = SPMV_K_PIPE;
            }
            if (R.spmv_kind == SPMV_K_TMAV) {
                if (R.n > 0) RC_TRY(build_sellv(h, R));
                else R.spmv_kind = SPMV_K_PLAIN;
            }
            if (R.spmv_kind != SPMV_K_TMA) {
                R.use_slots = false;
                R.n_explicit = R.nnz;
            }
        }
        if (multi(h)) RC_TRY(plan_split(h));
        RC_TRY(plan_start(h));
    }
    RC_TRY(stream_attrs());
    h->grid_md = grid_for((const void *)multidot_kernel<4, K_NP, K_NE, K_BS, U_MD4>, K_BS, h->nsm);
    h->small_grid = small_grid_for(h);
    CUDA_TRY(cudaStreamCreateWithFlags(&h->side, cudaStreamNonBlocking));
    CUDA_TRY(cudaStreamCreateWithFlags(&h->cstream, cudaStreamNonBlocking));
    for (auto &e : h->ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : h->evh) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : h->evc) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreate(&h->t0));
    CUDA_TRY(cudaEventCreate(&h->t1));
    CUDA_TRY(cudaMallocHost(&h->h_sc, sizeof(Scalars)));
    for (int i = 0; i < 2; ++i) {
        CUDA_TRY(cudaMallocHost(&h->h_poll[i], sizeof(Scalars)));
        CUDA_TRY(cudaEventCreateWithFlags(&h->evp[i], cudaEventDisableTiming));
    }
    *out = guard.release();
    return PBCG_OK;
}

extern "C" void pbicgstab_destroy(pbcg_handle *h) {
    if (!h) return;
    for (auto &g : h->gexec)
        if (g) cudaGraphExecDestroy(g);
    for (auto &e : h->ev)
        if (e) cudaEventDestroy(e);
    for (auto &e : h->evh)
        if (e) cudaEventDestroy(e);
    for (auto &e : h->evc)
        if (e) cudaEventDestroy(e);
    if (h->t0) cudaEventDestroy(h->t0);
    if (h->t1) cudaEventDestroy(h->t1);
    if (h->side) cudaStreamDestroy(h->side);
    if (h->cstream) cudaStreamDestroy(h->cstream);
    if (h->h_sc) cudaFreeHost(h->h_sc);
    for (int i = 0; i < 2; ++i) {
        if (h->h_poll[i]) cudaFreeHost(h->h_poll[i]);
        if (h->evp[i]) cudaEventDestroy(h->evp[i]);
    }
    if (h->comm_halo && g_nccl.CommDestroy) g_nccl.CommDestroy(h->comm_halo);
    if (h->comm_red && g_nccl.CommDestroy) g_nccl.CommDestroy(h->comm_red);
    delete h;
}

// ----------------------------------------------------------------------------
// vectors in/out (device or host pointers; virtual ranks: full vectors)
// ----------------------------------------------------------------------------
static bool is_host_ptr(const void *p) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeUnregistered;
}

static int scatter_in(pbcg_handle *h, const double *src, double *Rank::*dst_member, bool host) {
    for (auto &R : h->R) {
        const int64_t off = h->V > 1 ? R.rb : 0;
        CUDA_TRY(cudaMemcpyAsync(R.*dst_member, src + off, sizeof(double) * R.n,
                                 host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
    }
    return PBCG_OK;
}

// The own part of the SpMV input for the product "B u": u itself, or with the
// pipelined block Jacobi (R-25) u_hat = M^-1 u (bj_apply_kernel, the
// oracle's orc_bj_apply formula) -- the SpMV then computes A (M^-1 u).
static int own_to_pad(pbcg_handle *h, Rank &R, const double *src, int which) {
    if (R.pipe) {
        if (R.n == 0) return PBCG_OK;
        bj_apply_kernel<<<(int)std::min<int64_t>((R.n + 511) / 512, 4096), 256, 0, h->stream>>>(
            R.n, R.rb, R.ng, R.bji, src, padbuf(R, which) + R.own_off);
        CUDA_TRY(cudaGetLastError());
        return PBCG_OK;
    }
    if (src != padbuf(R, which) + R.own_off)
        CUDA_TRY(cudaMemcpyAsync(padbuf(R, which) + R.own_off, src, sizeof(double) * R.n, cudaMemcpyDeviceToDevice,
                                 h->stream));
    return PBCG_OK;
}

static int copy_own_to_pad(pbcg_handle *h, double *Rank::*src_member, int which) {
    for (auto &R : h->R) RC_TRY(own_to_pad(h, R, R.*src_member, which));
    return PBCG_OK;
}

// w (already the own part of wpad) as the SpMV input of t = B w
static int w_to_pad(pbcg_handle *h) {
    for (auto &R : h->R)
        if (R.pipe) RC_TRY(own_to_pad(h, R, R.w(), 1));
    return PBCG_OK;
}

static void opts_defaults(const pbcg_opts *o, pbcg_opts &e) {
    e.tol = 1e-10;
    e.max_iter = 10000;
    e.breakdown_eps = 1e-30;
    e.poll_every = 16;
    e.use_graphs = 1;
    e.dot_mode = PBCG_DOT_EXACT;
    e.method = PBCG_METHOD_PBICGSTAB;
    e.rr_period = 0;
    e.x0_zero = 0;
    e.range_mode = PBCG_RANGE_FULL;
    if (o) {
        e = *o;
        if (!(e.breakdown_eps > 0.0)) e.breakdown_eps = 1e-30;
        if (e.poll_every <= 0) e.poll_every = 16;
    }
}

// ----------------------------------------------------------------------------
// start / iterate / finish / solve
// ----------------------------------------------------------------------------
static int capture_chunk(pbcg_handle *h, int iters, int slot);
static bool small_on(const pbcg_handle *h);
static int start_alg1(pbcg_handle *h);
static int start_alg2_rest(pbcg_handle *h, bool r_is_b);
static int start_chunked(pbcg_handle *h, const double *b);
static int g_default_chunk = 16;

extern "C" int pbicgstab_start(pbcg_handle *h, const double *b, const double *x0, const pbcg_opts *o) {
    NvtxRange nvtx_("pbcg.start (I1-I4)");
    if (!h || h->comm_only) return fail(PBCG_EINVAL, "start: no matrix on this handle");
    pbcg_opts op;
    opts_defaults(o, op);
    if (!b || (!x0 && !op.x0_zero)) return fail(PBCG_EINVAL, "start: b and x0 (or x0_zero) are required");
    if (!(op.tol >= 0.0) || op.max_iter < 0) return fail(PBCG_EINVAL, "start: bad tol / max_iter");
    if (op.dot_mode != PBCG_DOT_EXACT && op.dot_mode != PBCG_DOT_PLAIN) return fail(PBCG_EINVAL, "start: bad dot_mode");
    if (op.method != PBCG_METHOD_PBICGSTAB && op.method != PBCG_METHOD_BICGSTAB)
        return fail(PBCG_EINVAL, "start: bad method");
    if (op.method == PBCG_METHOD_BICGSTAB && op.dot_mode != PBCG_DOT_EXACT)
        return fail(PBCG_EINVAL, "start: Algorithm 1 runs with exact dots only");
    if (op.rr_period < 0) return fail(PBCG_EINVAL, "start: rr_period < 0");
    if (op.method == PBCG_METHOD_BICGSTAB && h->precond == PBCG_PRECOND_BJACOBI2_PIPE)
        return fail(PBCG_EINVAL, "start: the pipelined block Jacobi is defined for Algorithm 2");
    if (op.range_mode != PBCG_RANGE_FULL && op.range_mode != PBCG_RANGE_FAST)
        return fail(PBCG_EINVAL, "start: bad range_mode");
    if (op.rr_period > 0 && op.method != PBCG_METHOD_PBICGSTAB)
        return fail(PBCG_EINVAL, "start: residual replacement is defined for Algorithm 2");
    h->max_iter = op.max_iter;
    h->dot_mode = op.dot_mode;
    h->method = op.method;
    h->rr_period = op.rr_period;
    h->it_enq = 0;
    Scalars s0{};
    s0.tol = op.tol;
    s0.eps = op.breakdown_eps;
    s0.max_iter = op.max_iter;
    s0.hist_cap = h->hist_cap;
    s0.status = ST_RUNNING;
    s0.range_mode = op.range_mode;
    for (auto &R : h->R) {
        CUDA_TRY(cudaMemsetAsync(R.gsm, 0, sizeof(long long) * 4 * (size_t)GW4, h->stream));
        CUDA_TRY(cudaMemsetAsync(R.gbar, 0, sizeof(unsigned) * 16, h->stream));
        CUDA_TRY(cudaMemcpyAsync(R.sc, &s0, sizeof(Scalars), cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(cudaMemsetAsync(R.hist, 0, sizeof(double) * (size_t)h->hist_cap * H_COLS, h->stream));
        CUDA_TRY(cudaMemsetAsync(R.bad, 0, sizeof(int) * 4, h->stream));
    }
    // x0 = 0 (x0_zero): r0 = b - A 0 is b bit for bit -- every row's fma
    // chain over +0 (or, after y0 = M x0, +-0) inputs is +0 since A is finite
    // (setup checks), and b - (+0) = b -- so the residual SpMV is skipped and
    // r, r^ are copies of b (I1).  A host b then streams in
    // chunks on the side stream, each chunk's NaN/Inf scan and copies on the
    // main stream behind it (the copy overlaps that work).
    const bool zero_start = op.x0_zero != 0;
    const bool chunked = zero_start && op.method == PBCG_METHOD_PBICGSTAB && is_host_ptr(b) && h->R.size() == 1 &&
                         !h->R[0].st_row.empty();
    if (chunked) {
        for (auto &R : h->R) CUDA_TRY(cudaMemsetAsync(R.x, 0, sizeof(double) * R.n, h->stream));
    } else if (zero_start) {
        const bool hostb = is_host_ptr(b);
        for (auto &R : h->R) {
            if (R.n == 0) continue;
            const int64_t off = h->V > 1 ? R.rb : 0;
            const int nch = (hostb && h->R.size() == 1 && R.n >= (1 << 20)) ? 8 : 1;
            const int64_t step = ((R.n + nch - 1) / nch + 63) / 64 * 64;
            if (nch > 1) {  // the side stream starts after everything enqueued so far
                CUDA_TRY(cudaEventRecord(h->ev[4], h->stream));
                CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev[4], 0));
            }
            for (int k = 0; k < nch; ++k) {
                const int64_t c0 = std::min<int64_t>(R.n, k * step), c1 = std::min<int64_t>(R.n, c0 + step);
                if (c1 <= c0) break;
                const size_t by = sizeof(double) * (size_t)(c1 - c0);
                if (nch > 1) {
                    CUDA_TRY(cudaMemcpyAsync(R.b + c0, b + off + c0, by, cudaMemcpyHostToDevice, h->side));
                    CUDA_TRY(cudaEventRecord(h->evc[k], h->side));
                    CUDA_TRY(cudaStreamWaitEvent(h->stream, h->evc[k], 0));
                } else {
                    CUDA_TRY(cudaMemcpyAsync(R.b + c0, b + off + c0, by,
                                             hostb ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, h->stream));
                }
                nonfinite_scan_kernel<<<(int)std::min<int64_t>((c1 - c0 + 255) / 256, 4096), 256, 0, h->stream>>>(
                    c1 - c0, R.b + c0, R.bad);
                CUDA_TRY(cudaGetLastError());
                CUDA_TRY(cudaMemcpyAsync(R.r + c0, R.b + c0, by, cudaMemcpyDeviceToDevice, h->stream));
                CUDA_TRY(cudaMemcpyAsync(R.rh + c0, R.b + c0, by, cudaMemcpyDeviceToDevice, h->stream));
            }
        }
        for (auto &R : h->R) CUDA_TRY(cudaMemsetAsync(R.x, 0, sizeof(double) * R.n, h->stream));
    } else {
        RC_TRY(scatter_in(h, b, &Rank::b, is_host_ptr(b)));
        RC_TRY(scatter_in(h, x0, &Rank::x, is_host_ptr(x0)));
    }
    if (h->precond == PBCG_PRECOND_BJACOBI2 || h->precond == PBCG_PRECOND_BJACOBI2_PIPE)  // y0 := M x0 (R-23, R-25)
        for (auto &R : h->R)
            if (R.n > 0) {
                bj_apply_kernel<<<(int)std::min<int64_t>((R.n + 511) / 512, 4096), 256, 0, h->stream>>>(
                    R.n, R.rb, h->n_global, R.bjm, R.x, R.x);
                CUDA_TRY(cudaGetLastError());
            }
    if (h->precond == PBCG_PRECOND_JACOBI)  // y0 := D x0 (R-22)
        for (auto &R : h->R)
            if (R.n > 0) {
                vec_muldiv_kernel<<<(int)std::min<int64_t>((R.n + 255) / 256, 4096), 256, 0, h->stream>>>(
                    R.n, R.x, R.dg, R.x, 0);
                CUDA_TRY(cudaGetLastError());
            }
    if (!zero_start) {
        for (auto &R : h->R) {
            if (R.n == 0) continue;
            const int grid = (int)std::min<int64_t>((R.n + 255) / 256, 4096);
            nonfinite_scan_kernel<<<grid, 256, 0, h->stream>>>(R.n, R.b, R.bad);
            nonfinite_scan_kernel<<<grid, 256, 0, h->stream>>>(R.n, R.x, R.bad);
            CUDA_TRY(cudaGetLastError());
        }
        // I1: r0 := b - A x0 ; r^ := r0 ; w0 := A r0 ; t0 := A w0   (R-1)
        RC_TRY(copy_own_to_pad(h, &Rank::x, 2));
        RC_TRY(halo(h, 2));
        for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_RESID, R.xpad, R.r, R.b, R.rh, false, h->stream));
    }
    if (h->method == PBCG_METHOD_BICGSTAB) RC_TRY(start_alg1(h));
    else if (chunked) RC_TRY(start_chunked(h, b));
    else RC_TRY(start_alg2_rest(h, zero_start));
    CUDA_TRY(cudaMemcpyAsync(h->h_sc, h->R[0].sc, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    int bad = 0;
    for (auto &R : h->R) {
        int bb = 0;
        CUDA_TRY(cudaMemcpy(&bb, R.bad, sizeof(int), cudaMemcpyDeviceToHost));
        bad |= bb;
    }
    h->started = true;
    if (bad & 2) return fail(PBCG_ENONFINITE, "start: NaN/Inf in b or x0");
    if (h->h_sc->err) return fail(PBCG_EINVAL, "start: ||b|| = 0");
    // capture the iteration graph now (nothing runs), so that the first
    // iterate()/solve() chunk does not pay for capture + instantiation
    h->chunk = o ? op.poll_every : g_default_chunk;
    if (op.use_graphs && h->stream && !small_on(h)) RC_TRY(capture_chunk(h, h->chunk, 0));
    return PBCG_OK;
}

// I1-I4 of Algorithm 2 from x0 = 0 with a host b, chunk by chunk (plan_start):
// chunk k of b lands (side stream) -> its scan and r = r^ = b copies; then
// w0 = A r0 over chunk k-1's rows (their x rows lie in chunks <= k), then
// t0 = A w0 over chunk k-2's rows and its share of (w0,b), (b,b) (the
// exact dots accumulate over the launches; the last one rounds: PH_INIT0).
// The same operations as start_alg2_rest, so the same bits.
static int start_chunked(pbcg_handle *h, const double *b) {
    Rank &R = h->R[0];
    const cudaStream_t st = h->stream;
    CUDA_TRY(cudaEventRecord(h->ev[4], st));  // the side stream starts after the memsets
    CUDA_TRY(cudaStreamWaitEvent(h->side, h->ev[4], 0));
    for (int k = 0; k < START_NCH; ++k) {
        const int64_t c0 = R.st_row[k], c1 = R.st_row[k + 1];
        CUDA_TRY(cudaMemcpyAsync(R.b + c0, b + c0, sizeof(double) * (size_t)(c1 - c0), cudaMemcpyHostToDevice, h->side));
        CUDA_TRY(cudaEventRecord(h->evc[k], h->side));
    }
    double *x2 = padbuf(R, 2) + R.own_off;  // the SpMV input of w0 = A r0
    for (int k = 0; k < START_NCH + 2; ++k) {
        if (k < START_NCH) {
            const int64_t c0 = R.st_row[k], c1 = R.st_row[k + 1];
            const size_t by = sizeof(double) * (size_t)(c1 - c0);
            CUDA_TRY(cudaStreamWaitEvent(st, h->evc[k], 0));
            nonfinite_scan_kernel<<<(int)std::min<int64_t>((c1 - c0 + 255) / 256, 4096), 256, 0, st>>>(c1 - c0, R.b + c0,
                                                                                                  R.bad);
            CUDA_TRY(cudaGetLastError());
            CUDA_TRY(cudaMemcpyAsync(R.r + c0, R.b + c0, by, cudaMemcpyDeviceToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(R.rh + c0, R.b + c0, by, cudaMemcpyDeviceToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(x2 + c0, R.b + c0, by, cudaMemcpyDeviceToDevice, st));
        }
        if (k >= 1 && k - 1 < START_NCH) {  // w0 = A r0 over chunk k-1
            const int j = k - 1;
            spmv_dispatch<SPMV_PLAIN>(h, R, padbuf(R, 2), R.w(), nullptr, nullptr, nullptr, st, R.st_u[j], R.st_u[j + 1], 0);
            CUDA_TRY(cudaGetLastError());
        }
        if (k >= 2) {  // t0 = A w0 over chunk k-2, and its share of the init dots
            const int m = k - 2;
            spmv_dispatch<SPMV_PLAIN>(h, R, padbuf(R, 1), R.t, nullptr, nullptr, nullptr, st, R.st_u[m], R.st_u[m + 1], 0);
            CUDA_TRY(cudaGetLastError());
            const int64_t c0 = R.st_row[m], c1 = R.st_row[m + 1];
            MultiDotArgs a{};
            a.n = c1 - c0;
            a.x[0] = R.w() + c0;
            a.y[0] = R.b + c0;
            a.x[1] = a.y[1] = R.b + c0;
            a.sc = R.sc;
            a.gacc = R.gacc[0];
            a.ticket = m == START_NCH - 1 ? R.tickets : nullptr;  // the last launch rounds
            a.hist = R.hist;
            a.phase = PH_INIT0;
            a.finalize = 1;
            RC_TRY(launch_xd2(h, a));
        }
    }
    return PBCG_OK;
}

// I1 (rest) - I4 of Algorithm 2.  r_is_b: r0 = r^ = b bit for bit (x0 = 0),
// so the dots read b for all three (the same values, fewer distinct bytes).
static int start_alg2_rest(pbcg_handle *h, bool r_is_b) {
    RC_TRY(copy_own_to_pad(h, &Rank::r, 2));
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, R.xpad, R.w(), nullptr, nullptr, false, h->stream));
    RC_TRY(w_to_pad(h));
    RC_TRY(halo(h, 1));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, padbuf(R, 1), R.t, nullptr, nullptr, false, h->stream));
    // I2-I4: ||b||, rho0 = (r^,r0), delta0 = (r^,w0), (r0,r0); alpha0
    std::vector<const double *> xb, yb, xr, yr, xw, yw, xn, yn;
    for (auto &R : h->R) {
        const double *r = r_is_b ? R.b : R.r, *rh = r_is_b ? R.b : R.rh;
        xb.push_back(R.b); yb.push_back(R.b);
        xr.push_back(rh); yr.push_back(r);
        xw.push_back(rh); yw.push_back(R.w());
        xn.push_back(r); yn.push_back(r);
    }
    if (r_is_b) {  // (w0, b) and (b, b) in one pass of the two-dot stream kernel (PH_INIT0)
        const double *const *xs[4] = {yw.data(), yb.data(), nullptr, nullptr};
        const double *const *ys[4] = {yb.data(), yb.data(), nullptr, nullptr};
        return multidot(h, 0, PH_INIT0, 2, xs, ys);
    }
    const double *const *xs[4] = {xb.data(), xr.data(), xw.data(), xn.data()};
    const double *const *ys[4] = {yb.data(), yr.data(), yw.data(), yn.data()};
    return multidot(h, 0, PH_INIT, 4, xs, ys);
}

// Algorithm 1 init: r^ := r0 (written with r0), p0 := r0;
// ||b||, rho0 = (r^,r0), (r0,r0)
static int start_alg1(pbcg_handle *h) {
    for (auto &R : h->R)
        CUDA_TRY(cudaMemcpyAsync(R.z(), R.r, sizeof(double) * R.n, cudaMemcpyDeviceToDevice, h->stream));
    std::vector<const double *> xb, xr, yr, xn;
    for (auto &R : h->R) {
        xb.push_back(R.b);
        xr.push_back(R.rh);
        yr.push_back(R.r);
        xn.push_back(R.r);
    }
    const double *const *xs[4] = {xb.data(), xr.data(), xn.data(), xn.data()};
    const double *const *ys[4] = {xb.data(), yr.data(), xn.data(), xn.data()};
    return multidot(h, 0, PH1_INIT, 4, xs, ys);
}

// One iteration of Algorithm 1 with exact dots, vectors
// p -> z buffer (padded, SpMV input), s -> s, q -> w buffer (padded), y -> y.
// Four reduction phases, each a multidot whose last CTA (single rank) or
// finalize (ranks) runs phase1_finalize; every kernel is predicated on done.
static int enqueue_alg1(pbcg_handle *h) {
    cudaStream_t st = h->stream;
    auto grid1 = [&](const Rank &R) { return (int)std::max<int64_t>(1, std::min<int64_t>((R.n + 255) / 256, 4 * h->nsm)); };
    auto ptrs = [&](double *Rank::*m) {
        std::vector<const double *> v;
        for (auto &R : h->R) v.push_back(R.*m);
        return v;
    };
    std::vector<const double *> vz, vw;
    for (auto &R : h->R) { vz.push_back(R.z()); vw.push_back(R.w()); }
    const auto vrh = ptrs(&Rank::rh), vs = ptrs(&Rank::s), vy = ptrs(&Rank::y), vr = ptrs(&Rank::r);
    RC_TRY(halo(h, 0));  // s := A p
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, R.zpad, R.s, nullptr, nullptr, true, st));
    {
        const double *const *xs[4] = {vrh.data(), nullptr, nullptr, nullptr};
        const double *const *ys[4] = {vs.data(), nullptr, nullptr, nullptr};
        RC_TRY(multidot(h, 1, PH1_DEN, 1, xs, ys));  // a := rho/(r^,s)
    }
    for (auto &R : h->R) a1_q_kernel<<<grid1(R), 256, 0, st>>>(R.n, R.r, R.s, R.w(), R.sc);
    CUDA_TRY(cudaGetLastError());
    {
        const double *const *xs[4] = {vw.data(), nullptr, nullptr, nullptr};
        RC_TRY(multidot(h, 2, PH1_QQ, 1, xs, xs));  // ||q||/||b|| <= tol?
    }
    for (auto &R : h->R) {
        a1_xconv_kernel<<<grid1(R), 256, 0, st>>>(R.n, R.x, R.z(), R.sc);
        a1_qclear_kernel<<<1, 1, 0, st>>>(R.sc);
    }
    CUDA_TRY(cudaGetLastError());
    RC_TRY(halo(h, 1));  // y := A q
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, R.wpad, R.y, nullptr, nullptr, true, st));
    {
        const double *const *xs[4] = {vw.data(), vy.data(), nullptr, nullptr};
        const double *const *ys[4] = {vy.data(), vy.data(), nullptr, nullptr};
        RC_TRY(multidot(h, 1, PH1_OM, 2, xs, ys));  // w := (q,y)/(y,y)
    }
    for (auto &R : h->R) a1_xr_kernel<<<grid1(R), 256, 0, st>>>(R.n, R.x, R.z(), R.w(), R.y, R.r, R.sc);
    CUDA_TRY(cudaGetLastError());
    {
        const double *const *xs[4] = {vrh.data(), vr.data(), nullptr, nullptr};
        const double *const *ys[4] = {vr.data(), vr.data(), nullptr, nullptr};
        RC_TRY(multidot(h, 2, PH1_R, 2, xs, ys));  // rho', relres, beta
    }
    for (auto &R : h->R) a1_p_kernel<<<grid1(R), 256, 0, st>>>(R.n, R.r, R.z(), R.s, R.sc);
    CUDA_TRY(cudaGetLastError());
    return PBCG_OK;
}

static int capture_chunk(pbcg_handle *h, int iters, int slot) {
    cudaGraphExec_t &gx = h->gexec[slot];
    if (gx && h->g_iters[slot] == iters && h->g_mode[slot] == h->dot_mode + 2 * h->method) return PBCG_OK;
    if (gx) { cudaGraphExecDestroy(gx); gx = nullptr; }
    cudaGraph_t g;
    CUDA_TRY(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeRelaxed));
    int rc = PBCG_OK;
    for (int k = 0; k < iters && rc == PBCG_OK; ++k) rc = enqueue_iteration(h);
    cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (rc != PBCG_OK) return rc;
    if (e != cudaSuccess) return fail(PBCG_ECUDA, "graph capture: %s", cudaGetErrorString(e));
    CUDA_TRY(cudaGraphInstantiate(&gx, g, 0));
    cudaGraphDestroy(g);
    h->g_iters[slot] = iters;
    h->g_mode[slot] = h->dot_mode + 2 * h->method;
    return PBCG_OK;
}

// Residual replacement (NEXT-2, R-21): r := b - A x; w := A r; s := A p;
// z := A s; t := A w.  The SpMVs are predicated on the device done flag, so a
// solve that has stopped is left as it is.
static int enqueue_replacement(pbcg_handle *h) {
    cudaStream_t st = h->stream;
    RC_TRY(copy_own_to_pad(h, &Rank::x, 2));
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_RESID, R.xpad, R.r, R.b, nullptr, true, st));
    RC_TRY(copy_own_to_pad(h, &Rank::r, 2));
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, R.xpad, R.w(), nullptr, nullptr, true, st));
    RC_TRY(copy_own_to_pad(h, &Rank::p, 2));
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, R.xpad, R.s, nullptr, nullptr, true, st));
    RC_TRY(copy_own_to_pad(h, &Rank::s, 2));
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, R.xpad, R.z(), nullptr, nullptr, true, st));
    RC_TRY(w_to_pad(h));
    RC_TRY(halo(h, 1));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_PLAIN, padbuf(R, 1), R.t, nullptr, nullptr, true, st));
    return PBCG_OK;
}

// Fused small-system kernel (csrc/small.cuh): single rank, exact or plain
// dots, Algorithm 2 without replacement, n <= SMALL_N_MAX rows, cooperative launch
// available.  PBCG_SMALL=0 turns it off (A/B runs, and the six-kernel path's
// own tests).
static constexpr int SMALL_BS = 256;
static constexpr int64_t SMALL_N_MAX = 1 << 14;  // tools/small_ab.py: fused 50-55K vs 36-38K iter/s up to 16K rows, slower from 32K
static int small_grid_for(pbcg_handle *h) {
    if (h->comm_only || h->V != 1 || h->comm || h->R.empty() || h->precond == PBCG_PRECOND_BJACOBI2_PIPE) return 0;
    const Rank &R = h->R[0];
    if (R.n == 0 || R.n > SMALL_N_MAX) return 0;
    int coop = 0, per_sm = 0;
    if (cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->dev) != cudaSuccess || !coop) return 0;
    // launch_small may pick any of the four instantiations (the register-
    // resident ones use more registers): the grid must be co-resident for all
    per_sm = 1 << 30;
    const void *kerns[] = {(const void *)pbcg_small_kernel<SMALL_BS, true>, (const void *)pbcg_small_kernel<SMALL_BS, false>,
                           (const void *)pbcg_small_reg_kernel<SMALL_BS, true>,
                           (const void *)pbcg_small_reg_kernel<SMALL_BS, false>};
    for (const void *k : kerns) {
        int b = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, SMALL_BS, 0) != cudaSuccess) return 0;
        per_sm = std::min(per_sm, b);
    }
    const int64_t gran = R.h_perm.empty() ? 32 : 256;  // small.cuh: CTA row ranges
    const int64_t windows = (R.n + gran - 1) / gran;
    // at most 64 CTAs: C1 ran 55.1K iter/s at 64, 53.9K at 128 (one barrier counter, fewer arrivals)
    int64_t g = std::min<int64_t>({windows, (int64_t)std::max(per_sm, 0) * h->nsm, (int64_t)64});
    if (const char *e = getenv("PBCG_SMALL_GRID")) g = std::max<int64_t>(1, std::min<int64_t>(g, atoi(e)));  // A/B runs
    return (int)g;
}
static bool small_on(const pbcg_handle *h) {
    const char *e = getenv("PBCG_SMALL");
    return !(e && e[0] == '0') && h->small_grid > 0 && h->method == PBCG_METHOD_PBICGSTAB && h->rr_period == 0;
}
// The cluster kernel (cluster.cuh): systems of at most CL x 256 rows that the
// register-resident fused kernel takes (rows not permuted, <= 8 nonzeros per
// row), as ONE cluster of CL = 16 CTAs (non-portable; 8 if 16 cannot be
// scheduled).  0: not available.  PBCG_CLUSTER=0 turns it off (A/B runs).
static constexpr int CLUSTER_BS = 256;
static int cluster_size_for(pbcg_handle *h) {
    const char *e = getenv("PBCG_CLUSTER");
    if (e && e[0] == '0') return 0;
    if (h->R.empty()) return 0;
    const Rank &R = h->R[0];
    if (!R.h_perm.empty() || R.max_len > 8 || R.n == 0) return 0;
    static int cached = -1;
    if (cached < 0) {
        cached = 0;
        for (int cl : {16, 8}) {
            const void *k = (const void *)pbcg_cluster_kernel<CLUSTER_BS, true>;
            const int dsm = (int)ClusterSmem<CLUSTER_BS>::BYTES;
            if (cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, dsm) != cudaSuccess ||
                cudaFuncSetAttribute((const void *)pbcg_cluster_kernel<CLUSTER_BS, false>,
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, dsm) != cudaSuccess) {
                cudaGetLastError();
                break;
            }
            if (cl > 8) {
                if (cudaFuncSetAttribute(k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess ||
                    cudaFuncSetAttribute((const void *)pbcg_cluster_kernel<CLUSTER_BS, false>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
                    cudaGetLastError();
                    continue;
                }
            }
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cl);
            cfg.blockDim = dim3(CLUSTER_BS);
            cfg.dynamicSmemBytes = ClusterSmem<CLUSTER_BS>::BYTES;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cl;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int nclu = 0;
            if (cudaOccupancyMaxActiveClusters(&nclu, k, &cfg) == cudaSuccess && nclu >= 1) {
                cached = cl;
                break;
            }
            cudaGetLastError();
        }
    }
    if (cached == 0) return 0;
    const int64_t nw = (R.n + 31) / 32;
    return 32 * ((nw + cached - 1) / cached) <= CLUSTER_BS ? cached : 0;
}

static int launch_small(pbcg_handle *h, int32_t iters) {
    Rank &R = h->R[0];
    SmallArgs a{};
    a.n = R.n;
    a.slice_off = R.slice_off;
    a.row_len = R.row_len;
    a.val = R.sval;
    a.col = R.scol;
    a.perm = R.h_perm.empty() ? nullptr : R.perm;
    a.x = R.x; a.r = R.r; a.rh = R.rh; a.p = R.p; a.s = R.s; a.q = R.q; a.y = R.y; a.t = R.t; a.v = R.v;
    a.z = R.z();
    a.w = R.w();
    a.zpad = R.zpad;
    a.wpad = R.wpad;
    a.gA[0] = R.gsm; a.gA[1] = R.gsm + GW4; a.gB[0] = R.gsm + 2 * GW4; a.gB[1] = R.gsm + 3 * GW4;
    a.bar = R.gbar;
    a.sc = R.sc;
    a.hist = R.hist;
    a.iters = iters;
    void *args[] = {&a};
    if (const int cl = cluster_size_for(h)) {  // one thread-block cluster (cluster.cuh)
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(cl);
        cfg.blockDim = dim3(CLUSTER_BS);
        cfg.dynamicSmemBytes = ClusterSmem<CLUSTER_BS>::BYTES;
        cfg.stream = h->stream;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (h->dot_mode == PBCG_DOT_PLAIN) CUDA_TRY(cudaLaunchKernelEx(&cfg, pbcg_cluster_kernel<CLUSTER_BS, false>, a));
        else CUDA_TRY(cudaLaunchKernelEx(&cfg, pbcg_cluster_kernel<CLUSTER_BS, true>, a));
        return PBCG_OK;
    }
    // register-resident rows (small.cuh) when rows are not permuted, every CTA
    // holds at most SMALL_BS rows and no row more than 8 nonzeros (C1)
    const int64_t nw = (R.n + 31) / 32;
    const bool reg = R.h_perm.empty() && R.max_len <= 8 && 32 * ((nw + h->small_grid - 1) / h->small_grid) <= SMALL_BS &&
                     !(getenv("PBCG_SMALL_REG") && getenv("PBCG_SMALL_REG")[0] == '0');
    const bool plain = h->dot_mode == PBCG_DOT_PLAIN;
    const void *k = reg ? (plain ? (const void *)pbcg_small_reg_kernel<SMALL_BS, false>
                                 : (const void *)pbcg_small_reg_kernel<SMALL_BS, true>)
                        : (plain ? (const void *)pbcg_small_kernel<SMALL_BS, false>
                                 : (const void *)pbcg_small_kernel<SMALL_BS, true>);
    CUDA_TRY(cudaLaunchCooperativeKernel(k, dim3(h->small_grid), dim3(SMALL_BS), args, 0, h->stream));
    return PBCG_OK;
}

static int iterate_impl(pbcg_handle *h, int32_t k, int chunk, bool graphs) {
    NvtxRange nvtx_("pbcg.iterate");
    if (small_on(h)) {  // the fused small-system kernel: one launch runs all k iterations (or stops when done)
        if (k > 0) RC_TRY(launch_small(h, k));
        h->it_enq += k;
        return PBCG_OK;
    }
    if (graphs && h->stream == nullptr) graphs = false;  // cannot capture the legacy stream
    while (k > 0) {
        // iterations until the next replacement boundary (all of k without replacement)
        int32_t run = k;
        if (h->rr_period > 0) run = std::min<int64_t>(k, h->rr_period - h->it_enq % h->rr_period);
        k -= run;
        while (run > 0) {
            if (graphs && run >= chunk) {
                RC_TRY(capture_chunk(h, chunk, 0));
                CUDA_TRY(cudaGraphLaunch(h->gexec[0], h->stream));
                run -= chunk;
                h->it_enq += chunk;
            } else if (graphs && h->rr_period == 0) {  // the remainder: one graph of its own length
                RC_TRY(capture_chunk(h, run, 1));
                CUDA_TRY(cudaGraphLaunch(h->gexec[1], h->stream));
                h->it_enq += run;
                run = 0;
            } else {
                RC_TRY(enqueue_iteration(h));
                run -= 1;
                h->it_enq += 1;
            }
        }
        if (h->rr_period > 0 && h->it_enq % h->rr_period == 0) RC_TRY(enqueue_replacement(h));
    }
    return PBCG_OK;
}

extern "C" int pbicgstab_iterate(pbcg_handle *h, int32_t k) {
    if (!h || !h->started) return fail(PBCG_EINVAL, "iterate before start");
    if (k < 0) return fail(PBCG_EINVAL, "iterate: k < 0");
    return iterate_impl(h, k, h->chunk, true);
}

static int true_residual(pbcg_handle *h) {
    RC_TRY(copy_own_to_pad(h, &Rank::x, 2));
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) RC_TRY(launch_spmv(h, R, SPMV_RESID, R.xpad, R.tmp, R.b, nullptr, false, h->stream));
    std::vector<const double *> xt;
    for (auto &R : h->R) xt.push_back(R.tmp);
    const double *const *xs[4] = {xt.data(), nullptr, nullptr, nullptr};
    const double *const *ys[4] = {xt.data(), nullptr, nullptr, nullptr};
    return multidot(h, 3, PH_TRUE, 1, xs, ys);
}

extern "C" int pbicgstab_finish(pbcg_handle *h, double *x, pbcg_result *res) {
    NvtxRange nvtx_("pbcg.finish (true residual)");
    if (!h || !h->started) return fail(PBCG_EINVAL, "finish before start");
    // the copy-out of x (and Jacobi's x := D^-1 y) runs on the side stream
    // while the true residual (which only reads x) runs on the main stream
    cudaStream_t xs = x ? h->side : h->stream;
    if (x) {
        CUDA_TRY(cudaEventRecord(h->ev[4], h->stream));
        CUDA_TRY(cudaStreamWaitEvent(xs, h->ev[4], 0));
        const bool host = is_host_ptr(x);
        for (auto &R : h->R) {
            const int64_t off = h->V > 1 ? R.rb : 0;
            const double *src = R.x;
            if ((h->precond == PBCG_PRECOND_BJACOBI2 || h->precond == PBCG_PRECOND_BJACOBI2_PIPE) && R.n > 0) {  // x := M^-1 y (R-23, R-25), into q
                bj_apply_kernel<<<(int)std::min<int64_t>((R.n + 511) / 512, 4096), 256, 0, xs>>>(
                    R.n, R.rb, h->n_global, R.bji, R.x, R.q);
                CUDA_TRY(cudaGetLastError());
                src = R.q;
            }
            if (h->precond == PBCG_PRECOND_JACOBI && R.n > 0) {  // x := D^-1 y (R-22), into q (free after the loop)
                vec_muldiv_kernel<<<(int)std::min<int64_t>((R.n + 255) / 256, 4096), 256, 0, xs>>>(R.n, R.x, R.dg,
                                                                                                  R.q, 1);
                CUDA_TRY(cudaGetLastError());
                src = R.q;
            }
            CUDA_TRY(cudaMemcpyAsync(x + off, src, sizeof(double) * R.n,
                                     host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, xs));
        }
    }
    if (h->h_sc->err == 0) RC_TRY(true_residual(h));
    hist_digest_kernel<<<1, 32, 0, h->stream>>>(h->R[0].hist, h->R[0].sc);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(h->h_sc, h->R[0].sc, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (xs != h->stream) CUDA_TRY(cudaStreamSynchronize(xs));
    if (res) {
        const Scalars &s = *h->h_sc;
        res->status = s.status == ST_RUNNING ? PBCG_MAXITER : s.status;
        res->iterations = s.it;
        res->relres_recursive = s.relres;
        res->relres_true = s.relres_true;
        res->history_rows = std::min(s.it + 1, h->hist_cap);
        res->loop_seconds = 0.0;
        res->digest = s.digest;
    }
    return PBCG_OK;
}

extern "C" int pbicgstab_solve(pbcg_handle *h, const double *b, double *x, const pbcg_opts *o, pbcg_result *res) {
    if (!h || h->comm_only) return fail(PBCG_EINVAL, "solve: no matrix on this handle");
    if (!x) return fail(PBCG_EINVAL, "solve: x is required (in: x0)");
    pbcg_opts op;
    opts_defaults(o, op);
    RC_TRY(pbicgstab_start(h, b, x, &op));
    float ms = 0.f;
    CUDA_TRY(cudaEventRecord(h->t0, h->stream));
    // Polls overlap the next chunk: chunk k+1 is enqueued before the host
    // waits for the scalars copied after chunk k, so the GPU never idles on
    // the round trip (iterations after done are device-side no-ops).
    // The last chunk is cut to max_iter (its own graph, kept like the full
    // chunk's): no trailing no-op iterations when the solve runs to max_iter.
    int done_iters = 0, k = 0;
    while (!h->h_sc->done && done_iters < op.max_iter) {
        const int chunk = op.poll_every, cnt = std::min(chunk, op.max_iter - done_iters);
        RC_TRY(iterate_impl(h, cnt, chunk, op.use_graphs != 0));
        done_iters += cnt;
        CUDA_TRY(cudaMemcpyAsync(h->h_poll[k & 1], h->R[0].sc, sizeof(Scalars), cudaMemcpyDeviceToHost, h->stream));
        CUDA_TRY(cudaEventRecord(h->evp[k & 1], h->stream));
        if (k > 0) {  // the previous chunk's scalars
            CUDA_TRY(cudaEventSynchronize(h->evp[(k - 1) & 1]));
            *h->h_sc = *h->h_poll[(k - 1) & 1];
        }
        ++k;
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (k > 0) *h->h_sc = *h->h_poll[(k - 1) & 1];
    CUDA_TRY(cudaEventRecord(h->t1, h->stream));
    CUDA_TRY(cudaEventSynchronize(h->t1));
    CUDA_TRY(cudaEventElapsedTime(&ms, h->t0, h->t1));
    RC_TRY(pbicgstab_finish(h, x, res));
    if (res) res->loop_seconds = ms * 1e-3;
    return PBCG_OK;
}

extern "C" int pbicgstab_history(pbcg_handle *h, double *out, int32_t max_rows, int32_t *rows) {
    if (!h || h->comm_only || !out) return fail(PBCG_EINVAL, "history: bad arguments");
    Scalars s;
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    CUDA_TRY(cudaMemcpy(&s, h->R[0].sc, sizeof(Scalars), cudaMemcpyDeviceToHost));
    int nrow = std::min(std::min(s.it + 1, h->hist_cap), std::max(0, max_rows));
    if (nrow > 0)
        CUDA_TRY(cudaMemcpy(out, h->R[0].hist, sizeof(double) * H_COLS * nrow, cudaMemcpyDeviceToHost));
    if (rows) *rows = nrow;
    return PBCG_OK;
}

extern "C" int pbicgstab_spmv(pbcg_handle *h, const double *x, double *y) {
    if (!h || h->comm_only || !x || !y) return fail(PBCG_EINVAL, "spmv: bad arguments");
    for (auto &R : h->R) {
        const int64_t off = h->V > 1 ? R.rb : 0;
        CUDA_TRY(cudaMemcpyAsync(R.xpad + R.own_off, x + off, sizeof(double) * R.n, cudaMemcpyDeviceToDevice, h->stream));
    }
    RC_TRY(halo(h, 2));
    for (auto &R : h->R) {
        const int64_t off = h->V > 1 ? R.rb : 0;
        RC_TRY(launch_spmv(h, R, SPMV_PLAIN, R.xpad, y + off, nullptr, nullptr, false, h->stream));
    }
    return PBCG_OK;
}

// ----------------------------------------------------------------------------
// standalone EXDOT and the plain baseline dot
// ----------------------------------------------------------------------------
struct Scratch {
    long long *gacc = nullptr;
    unsigned *ticket = nullptr;
    double *out = nullptr;
    int32_t *flags = nullptr;
    double *partials = nullptr;
    unsigned *pticket = nullptr;
    int grid1 = 0, gridp = 0;
};
static std::mutex g_scr_mu;
static Scratch g_scr[64];

static int scratch(Scratch **out) {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(g_scr_mu);
    Scratch &S = g_scr[dev & 63];
    if (!S.gacc) {
        int nsm = 148;
        CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
        S.grid1 = grid_for((const void *)multidot_kernel<1, K_NP, K_NE, K_BS, U_MD1>, K_BS, nsm);
        S.gridp = grid_for((const void *)plain_dot_kernel<K_BS>, K_BS, nsm);
        CUDA_TRY(cudaMalloc(&S.gacc, sizeof(long long) * XS_GW));
        CUDA_TRY(cudaMalloc(&S.ticket, 64));
        CUDA_TRY(cudaMalloc(&S.out, 64));
        CUDA_TRY(cudaMalloc(&S.flags, 64));
        CUDA_TRY(cudaMalloc(&S.partials, sizeof(double) * (S.gridp + 1)));
        CUDA_TRY(cudaMalloc(&S.pticket, 64));
        CUDA_TRY(cudaMemset(S.gacc, 0, sizeof(long long) * XS_GW));
        CUDA_TRY(cudaMemset(S.ticket, 0, 64));
        CUDA_TRY(cudaMemset(S.pticket, 0, 64));
        CUDA_TRY(cudaDeviceSynchronize());
    }
    *out = &S;
    return PBCG_OK;
}

extern "C" int exdot(pbcg_handle *h, int64_t n, const double *x, const double *y, double *result, int32_t *flags,
                     int on_device, void *stream) {
    NvtxRange nvtx_("pbcg.exdot");
    if (n < 0 || !result || (n > 0 && (!x || !y))) return fail(PBCG_EINVAL, "exdot: bad arguments");
    cudaStream_t st = (cudaStream_t)stream;
    Scratch *S = nullptr;
    RC_TRY(scratch(&S));
    double *out = on_device ? result : S->out;
    int32_t *ofl = (on_device && flags) ? flags : S->flags;
    if (!h || (h->V == 1 && !h->comm)) {
        MultiDotArgs a{};
        a.n = n;
        a.x[0] = x;
        a.y[0] = y;
        a.sc = nullptr;
        a.gacc = (h && !h->R.empty()) ? h->R[0].gacc[4] : S->gacc;
        a.ticket = (h && !h->R.empty()) ? h->R[0].tickets + 4 : S->ticket;
        a.phase = PH_EXDOT;
        a.finalize = 1;
        a.out = out;
        a.out_flags = ofl;
        if (((((uintptr_t)x) | ((uintptr_t)y)) & 15) == 0 && n > 0) {
            RC_TRY(stream_attrs());
            XDS<<<stream_grid(h, n, TileGeo<X_NCW, XD_PPT>::T), STREAM_THREADS, XD_SMEM, st>>>(a);
        } else {
            const int grid = std::max(1, std::min<int>(S->grid1, (int)((n / 2 + K_BS - 1) / K_BS)));
            multidot_kernel<1, K_NP, K_NE, K_BS, U_MD1><<<grid, K_BS, 0, st>>>(a);
        }
        CUDA_TRY(cudaGetLastError());
    } else {
        // distributed: each (virtual) rank reduces its slice, int64 allreduce, round once
        const int P = (int)h->R.size();
        for (int v = 0; v < P; ++v) {
            const int64_t lo = (h->V > 1) ? n * v / P : 0, hi = (h->V > 1) ? n * (v + 1) / P : n;
            MultiDotArgs a{};
            a.n = hi - lo;
            a.x[0] = x + lo;
            a.y[0] = y + lo;
            a.gacc = h->R[v].gacc[4];
            a.ticket = h->R[v].tickets + 4;
            a.phase = PH_EXDOT;
            a.finalize = 0;  // the last CTA leaves normalised words for the allreduce
            if (((((uintptr_t)a.x[0]) | ((uintptr_t)a.y[0])) & 15) == 0 && a.n > 0) {
                RC_TRY(stream_attrs());
                XDS<<<stream_grid(h, a.n, TileGeo<X_NCW, XD_PPT>::T), STREAM_THREADS, XD_SMEM, st>>>(a);
            } else {
                const int grid = std::max(1, std::min<int>(S->grid1, (int)(((hi - lo) / 2 + K_BS - 1) / K_BS)));
                multidot_kernel<1, K_NP, K_NE, K_BS, U_MD1><<<grid, K_BS, 0, st>>>(a);
            }
            CUDA_TRY(cudaGetLastError());
        }
        RC_TRY(reduce_finalize<1>(h, 4, PH_EXDOT, st, out, ofl));
    }
    if (on_device) return PBCG_OK;
    int32_t fl = 0;
    CUDA_TRY(cudaMemcpyAsync(result, S->out, sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(&fl, S->flags, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    if (flags) *flags = fl;
    if (fl & FLAG_NONFINITE) return fail(PBCG_ENONFINITE, "exdot: NaN/Inf input");
    // the full-range pass ran on every flagged CTA (single GPU or per rank):
    // the value is the exactly rounded sum; only an overflow is an error
    if ((fl & FLAG_RANGE) && !std::isfinite(*result)) return fail(PBCG_ERANGE, "exdot: the exact sum overflows binary64");
    return PBCG_OK;
}

extern "C" int pbcg_dot_plain(int64_t n, const double *x, const double *y, double *result, void *stream) {
    if (n < 0 || !result) return fail(PBCG_EINVAL, "dot_plain: bad arguments");
    Scratch *S = nullptr;
    RC_TRY(scratch(&S));
    const int grid = std::max(1, std::min<int>(S->gridp, (int)((n / 2 + K_BS - 1) / K_BS)));
    plain_dot_kernel<K_BS><<<grid, K_BS, 0, (cudaStream_t)stream>>>(n, x, y, S->partials, S->pticket, result);
    CUDA_TRY(cudaGetLastError());
    return PBCG_OK;
}

extern "C" const char *pbicgstab_last_error(void) { return g_err.c_str(); }

extern "C" int pbcg_nccl_unique_id(uint8_t *out128) {
    if (!out128) return fail(PBCG_EINVAL, "null");
    if (!nccl_available()) return fail(PBCG_ENCCL, "libnccl.so.2 could not be loaded");
    ncclUniqueId id;
    NCCL_TRY(g_nccl.GetUniqueId(&id));
    memcpy(out128, &id, sizeof(id));
    return PBCG_OK;
}

extern "C" int pbcg_abi_version(void) { return PBCG_ABI_VERSION; }

extern "C" int pbcg_exec_mode(const pbcg_handle *h, int32_t *mode) {
    if (!h || !mode) return fail(PBCG_EINVAL, "exec_mode: null argument");
    *mode = small_on(h) ? 1 : 0;
    return PBCG_OK;
}

// Per-kernel device time of k more iterations (single rank): direct launches
// bracketed by CUDA events on the handle's stream.  ms[0..3] = summed ms of
// K2, SpMV(v=Az), K3, SpMV(t=Aw).  Same kernels and arguments as iterate().
extern "C" int pbcg_profile_iterations(pbcg_handle *h, int32_t k, double *ms) {
    if (!h || !h->started || k < 1 || !ms) return fail(PBCG_EINVAL, "profile: bad arguments");
    if (multi(h)) return fail(PBCG_EINVAL, "profile: single-rank handles only");
    if (h->method != PBCG_METHOD_PBICGSTAB) return fail(PBCG_EINVAL, "profile: Algorithm 2 only");
    constexpr int NK = 6;  // K2, finalize A, SpMV z, K3, finalize B, SpMV w (serialised here)
    std::vector<cudaEvent_t> ev((size_t)(NK + 1) * k);
    for (auto &e : ev) CUDA_TRY(cudaEventCreate(&e));
    Rank &R = h->R[0];
    cudaStream_t st = h->stream;
    int rc = PBCG_OK;
    for (int i = 0; i < k && rc == PBCG_OK; ++i) {
        cudaEvent_t *e = &ev[(size_t)(NK + 1) * i];
        cudaEventRecord(e[0], st);
        rc = launch_k2(h, R, 0, st);
        cudaEventRecord(e[1], st);
        if (h->dot_mode == PBCG_DOT_PLAIN) rc = reduce_finalize<4>(h, 1, PH_A, st, nullptr, nullptr);
        else finalize_kernel<4><<<1, 128, 0, st>>>(R.gacc[1], PH_A, R.sc, R.hist, nullptr, nullptr);
        cudaEventRecord(e[2], st);
        if (rc == PBCG_OK) rc = launch_spmv(h, R, SPMV_PLAIN, padbuf(R, 0), R.v, nullptr, nullptr, true, st);
        cudaEventRecord(e[3], st);
        if (rc == PBCG_OK) rc = launch_k3(h, R, 0, st);
        cudaEventRecord(e[4], st);
        if (rc == PBCG_OK && h->dot_mode == PBCG_DOT_PLAIN) rc = reduce_finalize<3>(h, 2, PH_B, st, nullptr, nullptr);
        else if (h->dot_mode != PBCG_DOT_PLAIN) finalize_kernel<3><<<1, 128, 0, st>>>(R.gacc[2], PH_B, R.sc, R.hist, nullptr, nullptr);
        cudaEventRecord(e[5], st);
        if (rc == PBCG_OK) rc = launch_spmv(h, R, SPMV_PLAIN, padbuf(R, 1), R.t, nullptr, nullptr, true, st);
        cudaEventRecord(e[6], st);
    }
    cudaError_t se = cudaStreamSynchronize(st);
    for (int j = 0; j < NK; ++j) ms[j] = 0.0;
    for (int i = 0; i < k && rc == PBCG_OK && se == cudaSuccess; ++i)
        for (int j = 0; j < NK; ++j) {
            float t = 0.f;
            cudaEventElapsedTime(&t, ev[(size_t)(NK + 1) * i + j], ev[(size_t)(NK + 1) * i + j + 1]);
            ms[j] += t;
        }
    for (auto &e : ev) cudaEventDestroy(e);
    if (se != cudaSuccess) return fail(PBCG_ECUDA, "profile: %s", cudaGetErrorString(se));
    return rc;
}

// Copy an internal solver vector (this rank's rows; virtual ranks: all rows)
// to `out` (device or host): 0 b, 1 x, 2 r, 3 r^, 4 p, 5 s, 6 z, 7 q, 8 y,
// 9 w, 10 t, 11 v -- the oracle's numbering.  Synchronises the stream.
extern "C" int pbcg_get_vector(pbcg_handle *h, int32_t which, double *out) {
    if (!h || h->comm_only || !out || which < 0 || which > 11) return fail(PBCG_EINVAL, "get_vector: bad arguments");
    const bool host = is_host_ptr(out);
    for (auto &R : h->R) {
        double *tab[12] = {R.b, R.x, R.r, R.rh, R.p, R.s, R.z(), R.q, R.y, R.w(), R.t, R.v};
        const int64_t off = h->V > 1 ? R.rb : 0;
        CUDA_TRY(cudaMemcpyAsync(out + off, tab[which], sizeof(double) * R.n,
                                 host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, h->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return PBCG_OK;
}

// Diagnostic spill counters (non-zero only in a -DPBCG_DEBUG_COUNTERS build).
extern "C" int pbcg_spmv_format(pbcg_handle *h, int64_t *out8) {
    if (!h || !out8) return fail(PBCG_EINVAL, "spmv_format: null argument");
    if (h->comm_only) return fail(PBCG_EINVAL, "spmv_format: handle has no matrix");
    for (int i = 0; i < 8; ++i) out8[i] = 0;
    for (const auto &R : h->R) {
        const int64_t slots = R.use_slots ? R.nslices * SELL_RS : 0;
        out8[0] += R.n;
        out8[1] += R.nnz;
        out8[2] += R.sell_nnz;
        out8[3] += R.n_explicit;
        out8[4] += slots;
        if ((R.spmv_kind == SPMV_K_TMA || R.spmv_kind == SPMV_K_TMAV) && R.blob)  // the packed chunks read once, x once, y
            out8[5] += R.blob_bytes + 8 * (R.nchunks + 1) + 16 * R.n + (R.h_perm.empty() ? 0 : 4 * R.n);
        else
            out8[5] += 8 * R.nnz + 4 * R.n_explicit + 4 * slots + 4 * R.n + 8 * R.nslices + 16 * R.n +
                       (R.h_perm.empty() ? 0 : 4 * R.n);
        out8[6] = std::max<int64_t>(out8[6], R.max_len);
        out8[7] |= R.h_perm.empty() ? 0 : 1;
    }
    return PBCG_OK;
}

extern "C" int pbcg_debug_counters(uint64_t *out16, int32_t reset) {
    if (!out16) return fail(PBCG_EINVAL, "null");
    CUDA_TRY(cudaMemcpyFromSymbol(out16, g_dbg, sizeof(unsigned long long) * 16));
    if (reset) {
        unsigned long long z[16] = {};
        CUDA_TRY(cudaMemcpyToSymbol(g_dbg, z, sizeof(z)));
    }
    return PBCG_OK;
}

// Per-CTA phase timestamps of a -DPBCG_TIMELINE build (zeros otherwise):
// out = 3 kinds (K2, SpMV SELL-P, K3) x 256 CTAs x 8 uint64 (globaltimer ns).
extern "C" int pbcg_timeline(uint64_t *out, int32_t reset) {
    if (!out) return fail(PBCG_EINVAL, "null");
    CUDA_TRY(cudaMemcpyFromSymbol(out, g_tl, sizeof(unsigned long long) * 3 * 256 * 8));
    if (reset) {
        std::vector<unsigned long long> z(3 * 256 * 8, 0ull);
        CUDA_TRY(cudaMemcpyToSymbol(g_tl, z.data(), sizeof(unsigned long long) * z.size()));
    }
    return PBCG_OK;
}

// kernel tuning knobs for benchmarks (not part of the numerical contract)
extern "C" int pbcg_set_chunk(int32_t iters) {
    if (iters < 1) return fail(PBCG_EINVAL, "chunk < 1");
    g_default_chunk = iters;
    return PBCG_OK;
}
