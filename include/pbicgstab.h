/*
 * pbicgstab.h -- C ABI of the B200-native hot path of arXiv 2404.13216:
 * pipelined BiCGStab (p-BiCGStab, §2 Algorithm 2, l.60-86) whose
 * inner products are computed ExBLAS-style (§2 l.95: floating-point
 * expansions + long accumulator, "independent of data partitioning, order of
 * computations, thread scheduling, or reduction tree schemes").
 *
 * Library: paper_2404_13216_b200/libpbicgstab.so (sm_100a).  Plain pointers
 * and sizes only; no C++ or torch types cross this boundary.  No function
 * aborts or throws: each returns a pbcg_rc and leaves a thread-local message
 * for pbicgstab_last_error().
 *
 * Conventions used below
 *   EXDOT(u,v)  the binary64 nearest (ties-to-even) to the exact real
 *               sum_k u_k v_k.  Exact zero -> +0.0.
 *   NORM(u)     sqrt(EXDOT(u,u)) (IEEE sqrt, round-to-nearest).
 *   SpMV        y_i = +0.0; for k in row i in ascending column order:
 *               y_i = fma(a_ik, x_k, y_i)  (R-6).
 *   Algorithm 2 is implemented with the readings R-1..R-15 of DESIGN.md
 *   (w0 := A r0, scalar omega vs vector w, i=0 copies, FMA policy F, ...).
 *   "device"    = CUDA global memory of the current device; "host" = CPU.
 *
 * Threading: a handle is used by one host thread at a time.  Collective
 * calls (setup, solve, start/iterate/finish, spmv, distributed exdot) must be
 * made by every rank with consistent arguments, as with MPI.
 */
#ifndef PBICGSTAB_H
#define PBICGSTAB_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PBCG_ABI_VERSION 10

/* return codes of every entry point (never an abort across the ABI) */
enum pbcg_rc {
    PBCG_OK = 0,
    PBCG_EINVAL = 1,     /* bad argument / dimension mismatch, ||b|| = 0 (l.259) */
    PBCG_ECUDA = 2,      /* CUDA runtime error (message in pbicgstab_last_error) */
    PBCG_ENCCL = 3,      /* NCCL error or NCCL unavailable for nranks > 1 */
    PBCG_ENOMEM = 4,     /* workspace too small */
    PBCG_ENONFINITE = 5, /* NaN/Inf in an input */
    PBCG_ERANGE = 6      /* exdot: a product outside the exact zone (R-9) or overflow */
};

/* solve outcome (pbcg_result.status); an outcome is not an error */
enum pbcg_status {
    PBCG_CONVERGED = 0,       /* ||r_i||/||b|| <= tol (recursive residual, R-10) */
    PBCG_MAXITER = 1,
    PBCG_BREAKDOWN_INIT = 2,  /* (r0,w0) = 0 or alpha_0 not finite (l.67) */
    PBCG_BREAKDOWN_RHO = 3,   /* |(r0,r_{i+1})| <= thr (R-11) */
    PBCG_BREAKDOWN_OMEGA = 4, /* omega_i = 0 and not converged (R-12) */
    PBCG_BREAKDOWN_ALPHA = 5, /* |alpha denominator| <= thr or not finite (R-11) */
    PBCG_RANGE = 6,           /* range_mode FULL: a NaN/Inf operand or an overflowing dot; FAST: a product
                                 outside the fast zone (R-9, R-24) */
    PBCG_RUNNING = -1
};

/* One rank's contiguous block of rows of the square global matrix, CSR.
 * All three arrays are DEVICE pointers, borrowed only for the duration of
 * pbicgstab_workspace_size / pbicgstab_setup (they are converted into the
 * workspace; the caller may free them afterwards). */
typedef struct {
    int64_t n_global;         /* global order n (rows = columns) */
    int64_t row_begin;        /* this rank owns global rows [row_begin, row_end) */
    int64_t row_end;
    int64_t nnz_local;        /* row_ptr[row_end-row_begin] */
    const int32_t *row_ptr;   /* device, n_local+1 entries, row_ptr[0] = 0, non-decreasing */
    const int32_t *col_idx;   /* device, GLOBAL column ids in [0,n_global), strictly increasing per row */
    const double *values;     /* device, finite */
} pbcg_csr_local;

/* Distribution.  nranks > 1: one process per GPU, NCCL over NVLink; every rank
 * passes its own contiguous row block (rank r owns the r-th block of any
 * contiguous partition; blocks must tile [0,n) in rank order).
 * virtual_ranks > 1 (requires nranks == 1 and the FULL matrix): the library
 * splits the rows into that many balanced blocks and runs them
 * as separate ranks inside this process on this GPU (halo exchange and
 * superaccumulator allreduce done with device copies) -- a partition-invariance
 * test vehicle on a single GPU. */
typedef struct {
    int32_t rank;
    int32_t nranks;
    const uint8_t *nccl_uid;  /* host, 128 bytes from pbcg_nccl_unique_id() on rank 0, same on all ranks; NULL if nranks == 1 */
    int32_t virtual_ranks;    /* 0 or 1 = off */
    int32_t history_capacity; /* rows of per-iteration scalar history kept on device; 0 -> 10001 */
    int32_t comm_mode;        /* 0 = auto; 1 = use the NCCL dataflow even with nranks == 1 (a 1-rank
                                 communicator: halo no-ops, allreduce = identity) -- test vehicle for the
                                 multi-GPU code path on one GPU */
    int32_t precond;          /* PBCG_PRECOND_NONE (0) or PBCG_PRECOND_JACOBI (1): right Jacobi
                                 preconditioning (R-22) folded into the
                                 matrix at setup: A' = A D^-1 (one RN division per stored entry, D =
                                 diag(A), zero or missing diagonal -> PBCG_EINVAL); solves A' y = b with
                                 y0 = D x0 and returns x = D^-1 y.  Residuals (and history) are those of
                                 A' y = b, i.e. of A x = b in exact arithmetic.
                                 PBCG_PRECOND_BJACOBI2 (2): right 2x2 point-block Jacobi (R-23):
                                 M = the 2x2 diagonal blocks of A (global rows 2m, 2m+1; 1x1 for the last
                                 row when n is odd), B = A M^-1 stored explicitly (each row's pattern
                                 widened to whole column blocks); y0 = M x0, x = M^-1 y.  Every rank's
                                 first row must be even; a singular or non-finite block -> PBCG_EINVAL.
                                 PBCG_PRECOND_BJACOBI2_PIPE (3): the same M applied INSIDE the iteration
                                 (R-25): A is stored as given; K2 writes
                                 z_hat = M^-1 z and K3 w_hat = M^-1 w beside z and w, and the SpMVs compute
                                 v = A z_hat, t = A w_hat (every product of Algorithm 2 is A (M^-1 u)).
                                 y0 = M x0, x = M^-1 y.  Algorithm 2 only; the fused small kernel is off;
                                 pbicgstab_spmv computes A x. */
} pbcg_dist;

enum pbcg_precond { PBCG_PRECOND_NONE = 0, PBCG_PRECOND_JACOBI = 1, PBCG_PRECOND_BJACOBI2 = 2,
                    PBCG_PRECOND_BJACOBI2_PIPE = 3 };

/* Solver options (SPEC.md l.214-217 SolverConfig subset). */
typedef struct {
    double tol;               /* stop when ||r_{i+1}||/||b|| <= tol (>= 0; 0 never converges) */
    int32_t max_iter;         /* >= 0 */
    double breakdown_eps;     /* relative breakdown threshold, default 1e-30; <= 0 -> 1e-30.
                                 Algorithm 2: thr = max(eps NORM(r0) NORM(r'), 1e-300) for |rho'| and the
                                 alpha denominator (R-11).  Ignored by
                                 PBCG_METHOD_BICGSTAB, whose breakdowns are exact zeros (R-20). */
    int32_t poll_every;       /* iterations per CUDA-graph chunk / host poll; <= 0 -> 16 */
    int32_t use_graphs;       /* 1: replay captured CUDA graphs of poll_every iterations; 0: direct launches */
    int32_t dot_mode;         /* PBCG_DOT_EXACT (0, default): ExBLAS exactly rounded dots, reproducible;
                                 PBCG_DOT_PLAIN (1): plain fp64 per-iteration dots (per-thread fma chains,
                                 fixed warp tree, CTA and grid sums in order; across NCCL ranks an fp64
                                 allreduce) -- the paper's non-reproducible comparison arm (SURVEY §8(f)
                                 NEXT-1); bits depend on the launch geometry and the partition.
                                 Init / true-residual dots stay exact in both modes. */
    int32_t method;           /* PBCG_METHOD_PBICGSTAB (0, default): Algorithm 2;
                                 PBCG_METHOD_BICGSTAB (1): Algorithm 1, classic BiCGStab (l.39-54) with
                                 exact dots, four reduction phases per iteration, the arithmetic of the
                                 oracle's orc_bicgstab_dots (R-20); requires PBCG_DOT_EXACT.
                                 history rows: 4 omega, 5 rho, 7 rr, 8 relres, 9 beta, 10 alpha. */
    int32_t rr_period;        /* Algorithm 2 with residual replacement (p-BiCGStabRR; SURVEY
                                 §8(f) NEXT-2): after every rr_period-th iteration that leaves the solve
                                 running, r := b - A x, w := A r, s := A p, z := A s, t := A w (DESIGN.md
                                 R-21).  0 (default) = never. */
    int32_t x0_zero;          /* 1: start from x0 = 0 without reading x0 (x0 may be NULL in pbicgstab_start;
                                 in pbicgstab_solve x is then the output buffer only): no host->device copy
                                 of the initial guess, and no residual SpMV -- r0 = b - A 0 = b bit for bit
                                 (A is finite), so r0 and r^ are copies of b; a host b of >= 2^20 rows on
                                 one rank is copied in 16 chunks, the init work of each chunk (copies,
                                 w0 = A r0, t0 = A w0, its share of the init dots) overlapping the copy.  With NCCL ranks it
                                 must agree on every rank (it decides whether start exchanges an x halo).
                                 0 (default): x0 is read. */
    int32_t range_mode;       /* PBCG_RANGE_FULL (0, default): every Algorithm 2 dot is exact over the whole
                                 binary64 range (R-24):
                                 a CTA whose products leave the fast zone (|fl(xy)| < 2^-960 or >= 2^1000)
                                 corrects them into an extended accumulator (LSB 2^-2148); only a NaN/Inf
                                 operand or a dot whose exact value rounds to +-inf ends the solve with
                                 PBCG_RANGE.  PBCG_RANGE_FAST (1): any product outside the fast zone ends
                                 it with PBCG_RANGE (R-9, R-19).  Algorithm 1 keeps R-9. */
} pbcg_opts;

enum pbcg_range_mode { PBCG_RANGE_FULL = 0, PBCG_RANGE_FAST = 1 };

enum pbcg_dot_mode { PBCG_DOT_EXACT = 0, PBCG_DOT_PLAIN = 1 };
enum pbcg_method { PBCG_METHOD_PBICGSTAB = 0, PBCG_METHOD_BICGSTAB = 1 };

/* Solve result.  history row layout (12 doubles per row, row 0 = init, row
 * i+1 = iteration i), identical to the oracle's:
 *   0 theta=(q,y) 1 eta=(y,y) 2 sigma=(r0,s) 3 zeta=(r0,z) 4 omega
 *   5 rho=(r0,r) 6 delta=(r0,w) 7 rr=(r,r) 8 relres=sqrt(rr)/||b||
 *   9 beta 10 alpha (next) 11 reserved (0)                                   */
typedef struct {
    int32_t status;           /* enum pbcg_status */
    int32_t iterations;       /* completed iterations */
    double relres_recursive;  /* sqrt((r,r))/||b|| at the last completed iteration */
    double relres_true;       /* NORM(b - A x)/NORM(b) */
    double loop_seconds;      /* device time of the iteration loop (CUDA events) */
    int32_t history_rows;     /* rows available via pbicgstab_history */
    int32_t reserved;
    uint64_t digest;          /* fingerprint of the scalar trajectory: FNV-1a 64 over the
                                 per-row FNV-1a 64 hashes of history rows 0 .. history_rows-1, each row
                                 hashed over its 12 doubles' bit patterns as 64-bit words (offset basis
                                 0xcbf29ce484222325, prime 0x100000001b3).  Bit-identical trajectories --
                                 at any rank count, any partition -- give the same digest. */
} pbcg_result;

typedef struct pbcg_handle pbcg_handle;

/* Bytes of device workspace pbicgstab_setup needs for A (A == NULL: a
 * comm-only handle for distributed exdot).  Local (not collective); copies
 * row_ptr to the host. */
int pbicgstab_workspace_size(const pbcg_csr_local *A, const pbcg_dist *dist, size_t *bytes);

/* Build a solver handle.  `stream` is the caller's cudaStream_t (NULL = legacy
 * default stream) on which all work is ordered; `workspace` is caller-owned
 * device memory of >= workspace_bytes that must outlive the handle (the
 * library makes no cudaMalloc after setup).  Converts A to the internal
 * sliced-ELL layout, plans the halo exchange, creates the NCCL communicators
 * (nranks > 1, each limited to a few CTAs through ncclConfig_t.maxCTAs so that
 * they run beside the interior SpMV), scans A for NaN/Inf (-> PBCG_ENONFINITE).
 * Collective: with nranks > 1 every rank allgathers
 * (row_begin, row_end, column hull, pbcg_config_hash) and checks them with
 * pbcg_check_ranks; a mismatch returns PBCG_EINVAL on every rank.
 * A == NULL: a comm-only handle (any nranks) for the distributed exdot; each
 * rank then passes its own contiguous slice of x and y. */
int pbicgstab_setup(const pbcg_csr_local *A, const pbcg_dist *dist, void *stream, void *workspace,
                    size_t workspace_bytes, pbcg_handle **out);

/* Solve A x = b with Algorithm 2.  b_local/x_local hold this rank's rows
 * (virtual ranks: the full vectors) and may be DEVICE or HOST pointers
 * (host buffers are staged through the workspace inside the call: the
 * "end-to-end" path).  x_local: in = x0, out = x.  Host-synchronous on
 * return.  Breakdown / max-iter are outcomes in result->status with rc 0. */
int pbicgstab_solve(pbcg_handle *h, const double *b_local, double *x_local, const pbcg_opts *opts,
                    pbcg_result *result);

/* Stepping interface (used by solve, bench and tracing):
 *   start    lines I1-I4: r0 = b - A x0, r^ = r0, w0 = A r0, t0 = A w0, the
 *            four initial EXDOTs and alpha_0; synchronises once to report
 *            EINVAL (||b|| = 0) / ENONFINITE.
 *   iterate  enqueue k more iterations on the stream (asynchronous; iterations
 *            after convergence/breakdown are device-side no-ops).
 *   finish   synchronise, true residual, copy x out (device or host pointer),
 *            fill result. */
int pbicgstab_start(pbcg_handle *h, const double *b_local, const double *x0_local, const pbcg_opts *opts);
int pbicgstab_iterate(pbcg_handle *h, int32_t k);
int pbicgstab_finish(pbcg_handle *h, double *x_local, pbcg_result *result);

/* Copy up to max_rows rows (12 doubles each, layout above) of the scalar
 * history of the last start/solve to host memory `out`; *rows = rows copied.
 * Identical on every rank and every virtual rank. */
int pbicgstab_history(pbcg_handle *h, double *out, int32_t max_rows, int32_t *rows);

/* y = A x for this rank's rows (x_local, y_local: device, n_local each; the
 * halo is exchanged internally).  Stream-ordered, asynchronous.  Virtual
 * ranks: full vectors. */
int pbicgstab_spmv(pbcg_handle *h, const double *x_local, double *y_local);

/* EXDOT over n_local elements of device vectors x, y.  h == NULL: single
 * GPU; otherwise the handle's ranks each pass their slice and the
 * superaccumulators are allreduced (int64 sum) before the single rounding.
 * result_on_device = 1: `result` (1 double) and `flags` (1 int32, may be
 * NULL) are device pointers, the call is stream-ordered on `stream` and
 * returns PBCG_OK; = 0: host pointers, the call synchronises.
 * flags: bit 1 (2) = some input is NaN/Inf (PBCG_ENONFINITE); otherwise
 * bit 0 (1) = some nonzero product has |fl(x*y)| < 2^-960 or >= 2^1000
 * (R-9), i.e. lies outside the fast pass's exact zone.  Single GPU
 * (h NULL, or one rank without NCCL): the CTAs that met such a product
 * correct it in the full-range pass (exact 106-bit products, accumulator
 * down to 2^-2148), so the result is still the exactly
 * rounded sum and
 * the call returns PBCG_OK unless that sum overflows binary64 (+-inf,
 * PBCG_ERANGE).  Distributed handles (virtual ranks, NCCL ranks, comm-only
 * handles of any nranks) do the same per rank: the flagged CTAs' extended
 * words are summed across ranks with the fast words (int64) and rounded once.
 * When bit 1 is set, bit 0 is unspecified.  n_local = 0 gives +0.0
 * (SPEC.md l.69). */
int exdot(pbcg_handle *h, int64_t n_local, const double *x, const double *y, double *result, int32_t *flags,
          int result_on_device, void *stream);

/* Plain (non-reproducible, tree-ordered) fp64 dot -- the measurement
 * baseline of BASELINE.json ("within 2x of a plain fp64 dot").  result is a
 * device pointer; stream-ordered. */
int pbcg_dot_plain(int64_t n, const double *x, const double *y, double *result, void *stream);

/* Release the handle (communicators, events, graphs).  Workspace stays the
 * caller's. */
void pbicgstab_destroy(pbcg_handle *h);

/* Message of the last failing call on this thread ("" if none). */
const char *pbicgstab_last_error(void);

/* 128-byte NCCL unique id (rank 0 calls it; broadcast it to every rank). */
int pbcg_nccl_unique_id(uint8_t *out128);

int pbcg_abi_version(void);

/* ---- measurement hooks (not part of the numerical contract) -------------- */

/* Enqueue k more iterations of a started single-rank solve as direct launches
 * serialised on the handle's stream and bracketed by CUDA events, synchronise,
 * and return in ms[0..5] the summed device time of K2 (l.70-74 + phase-A dot
 * partials), finalize A (round, omega: l.76), SpMV v=Az (l.75), K3 (l.77-79 +
 * phase-B partials), finalize B (round, beta/alpha/stop: l.81-82) and SpMV
 * t=Aw (l.80).  (In iterate() the finalizes overlap the SpMVs.) */
int pbcg_profile_iterations(pbcg_handle *h, int32_t k, double *ms);

/* Iterations per captured CUDA-graph chunk used by pbicgstab_iterate (>= 1). */
int pbcg_set_chunk(int32_t iters);

/* Copy internal vector `which` (0 b, 1 x, 2 r, 3 r^, 4 p, 5 s, 6 z, 7 q,
 * 8 y, 9 w, 10 t, 11 v; this rank's rows, virtual ranks: all rows) to `out`
 * (device or host, n_local doubles).  Synchronises.  Tests and diagnostics. */
int pbcg_get_vector(pbcg_handle *h, int32_t which, double *out);

/* Stored SpMV format of this handle (all its ranks), 8 int64:
 * [0] rows, [1] nonzeros, [2] sliced-ELL entries incl. padding, [3] column ids
 * read explicitly (the rest follow from a per slice-slot offset: every row of
 * the 32-row slice finds its k-th nonzero at x index row + d, k < 15),
 * [4] slot-record words (16 per slice, 0 if unused), [5] algorithmic bytes of
 * one SpMV = 8 nnz + 4 [3] + 4 [4] + 4 rows (lengths) + 8 slices + 16 rows
 * (x once, y) (+ 4 rows sigma-permutation), [6] longest row, [7] 1 if rows
 * are sigma-sorted.  The fold of every row is the CSR fma chain regardless
 * (R-6).  Host-only, no synchronisation. */
int pbcg_spmv_format(pbcg_handle *h, int64_t *out8);

/* How pbicgstab_iterate runs the iterations of the solve started last on
 * this handle: *mode = 0: six kernels per iteration (K2, SpMV, K3, SpMV and
 * the two side-stream finalizes), replayed from CUDA graphs; 1: the fused
 * small-system kernel (single rank, n <= 16384 rows, exact or plain dots, Algorithm 2
 * without replacement), ONE cooperative launch per iterate
 * call.  PBCG_SMALL=0 in the environment disables the fused kernel.
 * Host-only. */
int pbcg_exec_mode(const pbcg_handle *h, int32_t *mode);

/* Spill counters of a -DPBCG_DEBUG_COUNTERS build (16 uint64; zeros in the
 * release build): [1] warp spill votes, [2] overflow-tier entries, [3]
 * superaccumulator deposits.  reset != 0 clears them. */
int pbcg_debug_counters(uint64_t *out16, int32_t reset);

/* Per-CTA phase timestamps of a -DPBCG_TIMELINE build (tools/timeline.py;
 * zeros in the release build): 3 kernels (K2, SELL-P SpMV, K3) x 256 CTAs x 8
 * uint64 globaltimer values; reset != 0 clears them. */
int pbcg_timeline(uint64_t *out, int32_t reset);

/* ---- host-only planning helpers (no GPU needed; CPU-testable) ------------ */

/* FNV-1a hash of the setup arguments every rank must agree on: ABI version,
 * n_global (-1 for a comm-only handle), nranks, virtual_ranks, precond,
 * comm_mode. */
int pbcg_config_hash(const pbcg_csr_local *A, const pbcg_dist *dist, uint64_t *out);

/* The check setup runs on the allgathered records, PBCG_RANK_REC int64 per
 * rank: (row_begin, row_end, cmin, cmax, config hash).  PBCG_EINVAL (with a
 * message naming the rank) if a hash differs from rank 0's or, with a
 * matrix, if the row blocks do not tile [0, n_global) in rank order. */
#define PBCG_RANK_REC 5
int pbcg_check_ranks(int32_t nranks, const int64_t *records, int64_t n_global, int32_t has_matrix);

/* pbcg_result.digest of a history held in host memory (rows x 12 doubles,
 * the layout of pbicgstab_history): the host twin of the device kernel, for
 * comparing trajectories saved from different runs.  rows >= 0. */
int pbcg_history_digest(const double *history, int32_t rows, uint64_t *out);

/* Balanced contiguous partition of n rows over p ranks (SPEC.md l.148,
 * l.185-187): the first n mod p ranks get one extra row.  begins: p+1 entries. */
int pbcg_plan_partition(int64_t n, int32_t p, int64_t *begins);

/* Halo plan for rank `me` given every rank's [row_begin,row_end) and the
 * inclusive column hull [cmin,cmax] of its local rows (ranges: 4*p int64,
 * cmax < cmin for a rank without nonzeros).  Outputs (p int64 each):
 *   recv_lo/recv_hi  global rows [lo,hi) this rank receives from rank q
 *   send_lo/send_hi  global rows [lo,hi) this rank sends to rank q
 * (empty: lo == hi).  The x-buffer of rank `me` covers [*buf_lo, *buf_hi). */
int pbcg_plan_halo(int32_t p, int32_t me, const int64_t *ranges, int64_t *recv_lo, int64_t *recv_hi,
                   int64_t *send_lo, int64_t *send_hi, int64_t *buf_lo, int64_t *buf_hi);

/* Host twin of the device superaccumulator (same source as the device
 * normalise/round; CPU tests of the cross-rank merge path).  words: SACC
 * words (pbcg_sacc_words(), int64, 32-bit digits, bit 0 = 2^-1074).
 *   accumulate  words := normalised sum of x_k*y_k (TwoProd split; R-9 zone)
 *   round       *out := RN-even(value(words)); PBCG_ERANGE on overflow */
int pbcg_sacc_words(void);
int pbcg_sacc_accumulate(int64_t n, const double *x, const double *y, int64_t *words);
int pbcg_sacc_round(const int64_t *words, double *out);

#ifdef __cplusplus
}
#endif
#endif /* PBICGSTAB_H */
