"""GPU parity of SpMV and of the whole p-BiCGStab trajectory against the
oracle (BASELINE.json north_star: "The full p-BiCGStab iterate trajectory must
be bit-exact against the oracle and identical at 1/2/4/8 GPUs")."""
import struct

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def pb():
    import torch
    assert torch.cuda.is_available()
    import paper_2404_13216_b200 as pb
    return pb


def solver(pb, A, **kw):
    return pb.Solver(A.row_ptr, A.col, A.val, A.n, **kw)


def gpu_b(pb, S, A):
    """b := A*ones with the GPU SpMV (stencils), or the generated b."""
    import torch
    if A.rhs == "given":
        return torch.from_numpy(A.b).cuda()
    return S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))


# ------------------------------------------------------------------- SpMV ---

@pytest.mark.parametrize("name", ["c1_2d64", "small3d", "rand", "dense", "c3_3d128"])
def test_spmv_bitwise(pb, name):
    import torch
    A = {"c1_2d64": lambda: gen.make_config("c1_2d64"),
         "small3d": lambda: gen.stencil(3, 21, 100.0),
         "rand": lambda: gen.random_banded(50_001, seed=3, band=2000),
         "dense": lambda: gen.dense_as_sparse(97, seed=4, density=0.3),
         "c3_3d128": lambda: gen.make_config("c3_3d128")}[name]()
    S = solver(pb, A)
    for seed in (1, 2):
        x = gen.loguniform(A.n, seed, -20, 20)
        y = S.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(u64(y), u64(oracle.spmv(A, x))), name
    ones = S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda")).cpu().numpy()
    assert np.array_equal(u64(ones), u64(oracle.spmv(A, np.ones(A.n))))
    S.close()


def test_spmv_virtual_ranks(pb):
    import torch
    A = gen.random_banded(30_000, seed=8, band=3000)
    x = gen.uniform(A.n, 5)
    want = u64(oracle.spmv(A, x))
    for V in (2, 3, 8):
        S = solver(pb, A, virtual_ranks=V)
        y = S.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.array_equal(u64(y), want), V
        S.close()


def test_spmv_empty_rows_and_signed_zero(pb):
    import torch
    A = gen.CSR(40, np.array([0] + [1] * 20 + [2] * 20, np.int32), np.array([0, 39], np.int32),
                np.array([1.0, -1.0]))
    S = solver(pb, A)
    x = np.zeros(40)
    x[0] = -0.0
    y = S.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
    assert np.array_equal(u64(y), u64(oracle.spmv(A, x)))
    S.close()


def test_setup_rejects_bad_csr(pb):
    A = gen.from_dense(np.eye(4))
    bad = gen.CSR(4, A.row_ptr.copy(), A.col.copy(), A.val.copy())
    bad.val[2] = np.nan
    with pytest.raises(pb.PbcgError) as e:
        solver(pb, bad)
    assert e.value.rc == 5
    bad = gen.CSR(4, np.array([0, 2, 3, 4, 5], np.int32), np.array([1, 0, 2, 3, 3], np.int32), np.ones(5))
    with pytest.raises(pb.PbcgError) as e:
        solver(pb, bad)
    assert e.value.rc == 1


# ------------------------------------------------------------- trajectory ---

def run_both(pb, A, tol, max_iter, steps=None, **kw):
    import torch
    S = solver(pb, A, history_capacity=max_iter + 1, **{k: v for k, v in kw.items() if k in ("virtual_ranks", "force_nccl")})
    b = gpu_b(pb, S, A)
    O = oracle.PBiCGStab(A, b=None if A.rhs != "given" else A.b, tol=tol, max_iter=max_iter)
    assert O.rc == 0
    assert np.array_equal(u64(b.cpu().numpy()), u64(O.vec("b")))
    O.run(steps)
    if steps is None:
        x, r = S.solve(b, tol=tol, max_iter=max_iter, poll_every=kw.get("poll_every", 16),
                       use_graphs=kw.get("use_graphs", True))
    else:
        S.start(b, tol=tol, max_iter=max_iter)
        S.iterate(steps)
        x = torch.zeros(A.n_local if hasattr(A, "n_local") else A.n, dtype=torch.float64, device="cuda")
        r = S.finish(x)
    H = S.history()
    S.close()
    return S, O, x.cpu().numpy(), r, H


def trajectory_digest(H):
    """pbcg_result.digest (include/pbicgstab.h) of a history array, written
    out: FNV-1a 64 over the per-row FNV-1a 64 hashes of the rows' bits."""
    B, P, M = 0xcbf29ce484222325, 0x100000001b3, (1 << 64) - 1
    h = B
    for row in u64(np.atleast_2d(H)):
        rh = B
        for w in row:
            rh = ((rh ^ int(w)) * P) & M
        h = ((h ^ rh) * P) & M
    return h


def assert_same(O, x, r, H, A):
    Ho = O.history()
    assert r.digest == trajectory_digest(Ho)  # the trajectory fingerprint of the oracle's history
    assert r.iterations == O.iterations, (r.iterations, O.iterations)
    st = O.status if O.status != oracle.RUNNING else oracle.MAXITER
    assert r.status == st, (r.status, O.status)
    assert H.shape == Ho.shape
    bad = np.argwhere(u64(H) != u64(Ho))
    assert bad.size == 0, f"first differing (row, col): {bad[:5].tolist()} gpu={H[tuple(bad[0])]!r} oracle={Ho[tuple(bad[0])]!r}"
    assert np.array_equal(u64(x), u64(O.vec("x")))


def test_c1_to_convergence(pb):
    # BASELINE.json configs[0], full trajectory, final x bits, true residual
    A = gen.make_config("c1_2d64")
    S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=500)
    assert r.status == pb.CONVERGED
    assert_same(O, x, r, H, A)
    tr, _ = oracle.true_relres(A, O.vec("b"), O.vec("x"))
    assert struct.pack("<d", r.relres_true) == struct.pack("<d", tr)
    # north_star: agrees with a plain-double BiCGStab within 1e-10
    st, it, xb, _ = oracle.bicgstab(A, O.vec("b"), tol=1e-10, max_iter=500)
    assert st == oracle.CONVERGED
    assert abs(r.relres_true - oracle.true_relres(A, O.vec("b"), xb)[0]) <= 1e-10


@pytest.mark.parametrize("V", [2, 3, 4, 8])
def test_c1_virtual_ranks_identical(pb, V):
    A = gen.make_config("c1_2d64")
    S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=500, virtual_ranks=V)
    assert_same(O, x, r, H, A)


def test_graphs_and_chunking_do_not_change_bits(pb):
    A = gen.stencil(3, 20, 100.0)
    ref = None
    for use_graphs, poll in [(True, 16), (False, 1), (True, 7)]:
        S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=2000, use_graphs=use_graphs, poll_every=poll)
        assert_same(O, x, r, H, A)
        if ref is None:
            ref = (x, H)
        assert np.array_equal(u64(ref[0]), u64(x)) and np.array_equal(u64(ref[1]), u64(H))


def test_small3d_and_random_to_convergence(pb):
    for A in (gen.stencil(3, 24, 100.0), gen.random_banded(20_000, seed=9, band=1500)):
        S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=3000)
        assert r.status == pb.CONVERGED, A.name
        assert_same(O, x, r, H, A)


@pytest.mark.parametrize("name,steps", [("c3_3d128", 6), ("c4_small", 4)])
def test_full_size_first_iterations(pb, name, steps):
    # full-size configs: first K iterations bit-exact plus the state after them
    A = gen.make_config("c3_3d128") if name == "c3_3d128" else gen.random_banded(1 << 19, seed=42)
    S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=10000, steps=steps)
    assert r.iterations == steps
    assert_same(O, x, r, H, A)


@pytest.mark.parametrize("V", [1, 3])
def test_wide_exponent_spread_takes_the_drain_fallback(pb, V):
    # A diagonal system whose entries span 2^-150 .. 2^150 (shuffled): w0 = A r0, t0 = A w0 and y = w - alpha z
    # spread the products of (y,y) over ~600 binades inside every warp, more than the 16-word window of the
    # end-of-kernel drain (exblas.cuh warp_window_deposit), so K2 / K3 take its per-term fallback; every dot is
    # still the exact sum rounded once, whatever the drain path or the rank count.
    n = 40_000  # above the fused small-system kernel's 16,384 rows: the six-kernel path
    e = np.floor(np.linspace(-150, 150, n)).astype(int)[np.random.default_rng(7).permutation(n)]
    d = np.ldexp(1.0 + gen.uniform(n, 9, 0.0, 1.0), e)
    A = gen.CSR(n, np.arange(n + 1, dtype=np.int32), np.arange(n, dtype=np.int32), d, name="diag_wide", rhs="given",
                b=gen.uniform(n, 10, 0.5, 1.5))
    S, O, x, r, H = run_both(pb, A, 0.0, 4, steps=4, virtual_ranks=V)
    assert_same(O, x, r, H, A)
    y = O.vec("y")
    assert np.log2(np.abs(y)).max() - np.log2(np.abs(y[y != 0])).min() > 280  # (y,y) spans > 560 bits: wider than the window


def test_diag2_and_breakdowns(pb):
    import torch
    # 1x1 diag(2), b = [2] -> one step, x = [1]
    A = gen.from_dense(np.array([[2.0]]))
    S = solver(pb, A)
    x, r = S.solve(torch.tensor([2.0], dtype=torch.float64, device="cuda"), tol=1e-10, max_iter=10)
    assert r.status == pb.CONVERGED and r.iterations == 1 and x.item() == 1.0
    S.close()
    # breakdown at init: (r0, A r0) = 0
    A = gen.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    S = solver(pb, A)
    x, r = S.solve(torch.tensor([1.0, 0.0], dtype=torch.float64, device="cuda"), tol=1e-10, max_iter=10)
    assert r.status == pb.BREAKDOWN_INIT and r.iterations == 0
    # ||b|| = 0 -> EINVAL; NaN in b -> ENONFINITE
    with pytest.raises(pb.PbcgError) as e:
        S.solve(torch.zeros(2, dtype=torch.float64, device="cuda"))
    assert e.value.rc == 1
    with pytest.raises(pb.PbcgError) as e:
        S.solve(torch.tensor([1.0, float("nan")], dtype=torch.float64, device="cuda"))
    assert e.value.rc == 5
    S.close()


def test_random_small_systems_match_oracle(pb):
    for k in range(12):
        n = 4 + 5 * k
        A = gen.dense_as_sparse(n, seed=100 + k, density=0.5)
        A.rhs = "given"
        A.b = gen.uniform(n, 200 + k)
        S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=500)
        assert_same(O, x, r, H, A)


def test_host_buffers_end_to_end(pb):
    # the e2e path: host b/x through the C ABI (staged inside the call)
    import torch
    A = gen.make_config("c1_2d64")
    S = solver(pb, A)
    b = S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
    xd, rd = S.solve(b, tol=1e-10, max_iter=500)
    xh, rh = S.solve(b.cpu().numpy(), tol=1e-10, max_iter=500)
    assert isinstance(xh, np.ndarray)
    assert rd.iterations == rh.iterations and np.array_equal(u64(xd.cpu().numpy()), u64(xh))
    S.close()


def test_nccl_dataflow_single_rank(pb):
    # The multi-GPU code path (K2/K3 publish -> int64 ncclAllReduce on the side
    # stream -> finalize_kernel; ncclSend/Recv halo) run on one GPU with a
    # 1-rank NCCL communicator, inside the CUDA graphs: identical bits.
    A = gen.make_config("c1_2d64")
    S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=500, force_nccl=True)
    assert_same(O, x, r, H, A)
    A = gen.random_banded(30_000, seed=17, band=2500)
    S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=400, force_nccl=True)
    assert_same(O, x, r, H, A)
    # 2x2 block Jacobi through the same path (its setup exchanges the columns
    # of M^-1 with the NCCL halo)
    B, M, Mi = oracle.block_jacobi_right(A)
    O = oracle.PBiCGStab(B, b=A.b, tol=1e-10, max_iter=400)
    O.run()
    S = solver(pb, A, history_capacity=401, force_nccl=True, precond="bjacobi2")
    import torch
    x, r = S.solve(torch.from_numpy(A.b).cuda(), tol=1e-10, max_iter=400)
    assert r.iterations == O.iterations and np.array_equal(u64(S.history()), u64(O.history()))
    assert np.array_equal(u64(x.cpu().numpy()), u64(oracle.bj_apply(Mi, O.vec("x"))))
    S.close()


def banded_with_holes(n, half, seed, holes_per_slice=0.3):
    """Band matrix |i-j| <= half with off-diagonal entries dropped at random
    (about `holes_per_slice` per 32 rows): slices mix uniform and explicit
    slot offsets."""
    rng = np.random.default_rng(seed)
    drop = holes_per_slice / (32 * (2 * half + 1))
    rows, cols = [], []
    for k in range(-half, half + 1):
        i = np.arange(max(0, -k), min(n, n - k))
        keep = (k == 0) | (rng.random(i.size) >= drop)
        rows.append(i[keep])
        cols.append(i[keep] + k)
    r = np.concatenate(rows)
    c = np.concatenate(cols)
    o = np.lexsort((c, r))
    r, c = r[o], c[o]
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, r + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    val = gen.loguniform(r.size, seed + 1, -3, 3)
    return gen.CSR(n, rp, c.astype(np.int32), val)


@pytest.mark.parametrize("kind", ["stencil3d", "band7", "band21"])
def test_spmv_slot_offsets(pb, kind, monkeypatch):
    # index compression of the sliced ELL (pbcg_spmv_format): per slice-slot
    # column offsets replace most column ids; identical bits with and without
    # them, for every SpMV kernel (TMA ring, register pipeline, row per thread)
    import torch
    A = {"stencil3d": lambda: gen.stencil(3, 96, 100.0),
         "band7": lambda: banded_with_holes(70_001, 3, 5),
         "band21": lambda: banded_with_holes(70_001, 10, 6)}[kind]()
    x = gen.loguniform(A.n, 3, -20, 20)
    xt = torch.from_numpy(x).cuda()
    want = u64(oracle.spmv(A, x))
    fmt = {}
    for kern in ("tma", "pipe", "plain"):
        monkeypatch.setenv("PBCG_SPMV_KERNEL", kern)
        for slots in ("1", "0"):
            monkeypatch.setenv("PBCG_SELL_SLOTS", slots)
            S = solver(pb, A)
            fmt[kern, slots] = f = S.spmv_format()
            assert f["rows"] == A.n and f["nnz"] == A.row_ptr[-1]
            assert np.array_equal(u64(S.spmv(xt).cpu().numpy()), want), (kern, slots)
            S.close()
    short_rows = int(np.diff(A.row_ptr).max()) <= 8
    for key, f in fmt.items():
        if key == ("tma", "1") and short_rows:
            # packed SELL-P chunks with slot records (the TMA kernel)
            assert 0 < f["explicit_cols"] < f["nnz"] // 2, f
            assert f["slot_records"] == 16 * ((A.n + 31) // 32)
            assert f["bytes_per_spmv"] < fmt["tma", "0"]["bytes_per_spmv"]
        else:  # every column id stored (plain / pipe kernels, long rows, slots off)
            assert f["explicit_cols"] == f["nnz"] and f["slot_records"] == 0, (key, f)
    # partitions: the records are per rank (offsets relative to each rank's buffer)
    monkeypatch.delenv("PBCG_SELL_SLOTS")
    monkeypatch.delenv("PBCG_SPMV_KERNEL")
    S = solver(pb, A, virtual_ranks=3)
    assert np.array_equal(u64(S.spmv(xt).cpu().numpy()), want)
    S.close()


def test_spmv_format_random_keeps_explicit(pb):
    # random banded rows (C4-like): no slot shares an offset, the plain kernels run
    A = gen.random_banded(40_000, seed=11, band=3000)
    S = solver(pb, A)
    f = S.spmv_format()
    assert f["explicit_cols"] == f["nnz"] and f["slot_records"] == 0 and f["sigma_sorted"] == 1
    S.close()


def ragged_long_rows(n, seed, lmax=255, wide_block=0, band=4000):
    """Rows of 0..lmax nonzeros (uniform lengths, some empty), columns inside
    +-band of the diagonal, loguniform values; rows [100, 100 + wide_block)
    get lmax nonzeros (slices wider than a SELL-V chunk's byte budget)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, lmax + 1, n)
    lens[rng.random(n) < 0.05] = 0
    lens[100:100 + wide_block] = lmax
    rp = np.zeros(n + 1, np.int64)
    cols = []
    for i in range(n):
        lo, hi = max(0, i - band), min(n, i + band + 1)
        c = np.unique(rng.integers(lo, hi, 2 * int(lens[i])))[:int(lens[i])]
        cols.append(c)
        rp[i + 1] = rp[i] + c.size
    col = np.concatenate(cols).astype(np.int32)
    val = gen.loguniform(col.size, seed + 1, -3, 3)
    return gen.CSR(n, rp.astype(np.int32), col, val, name=f"ragged{n}_{lmax}")


@pytest.mark.parametrize("kind", ["rand", "ragged60", "ragged200", "over255", "unbanded"])
def test_spmv_sellv(pb, kind, monkeypatch):
    # the TMA-streamed SELL-V kernel (long rows, padding-free byte-bounded
    # chunks, x window in shared memory): same bits as the oracle and as the
    # row-per-thread kernel, for ragged lengths, empty rows, a ragged tail
    # (n % 32 != 0), runs shorter than the ring, slices too wide for a deep
    # ring (ragged200: the matrix is loaded by the consumers, only chunk
    # headers pass through the ring).  Matrices it does not take fall back to
    # the row-per-thread kernel: rows over 255 nonzeros, x windows wider than
    # shared memory (unbanded)
    import torch
    A = {"rand": lambda: gen.random_banded(50_001, seed=3, band=2000),
         "ragged60": lambda: ragged_long_rows(20_011, 5, lmax=60, band=1000),
         "ragged200": lambda: ragged_long_rows(9_001, 6, lmax=200, wide_block=96, band=1000),
         "over255": lambda: ragged_long_rows(4_003, 7, lmax=300, wide_block=40),
         "unbanded": lambda: ragged_long_rows(60_007, 8, lmax=20, band=60_007)}[kind]()
    x = gen.loguniform(A.n, 3, -20, 20)
    xt = torch.from_numpy(x).cuda()
    want = u64(oracle.spmv(A, x))
    fmts = {}
    for kern in ("tmav", "plain"):
        monkeypatch.setenv("PBCG_SPMV_KERNEL", kern)
        for V in (1, 3):
            S = solver(pb, A, virtual_ranks=V)
            fmts[kern, V] = S.spmv_format()
            assert np.array_equal(u64(S.spmv(xt).cpu().numpy()), want), (kern, V)
            S.close()
    nnz = int(A.row_ptr[-1])
    f, fp = fmts["tmav", 1], fmts["plain", 1]
    assert f["explicit_cols"] == nnz and f["slot_records"] == 0
    if kind in ("over255", "unbanded"):
        assert f["bytes_per_spmv"] == fp["bytes_per_spmv"]  # the row-per-thread kernel ran
    else:
        # the chunks hold the nonzeros only (no ELL padding): about 12 B each
        assert f["bytes_per_spmv"] != fp["bytes_per_spmv"]
        assert 12 * nnz <= f["bytes_per_spmv"] - 16 * A.n <= 12 * nnz + 64 * (A.n // 32 + 1) + 8 * A.n


@pytest.mark.parametrize("V", [1, 3])
def test_sellv_solver_matches_oracle(pb, V, monkeypatch):
    # whole trajectories with the SELL-V SpMV (also under the virtual-rank
    # halo split: interior chunks, then the boundary ones)
    monkeypatch.setenv("PBCG_SPMV_KERNEL", "tmav")
    A = gen.random_banded(20_000, seed=9, band=1500)
    S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=3000, virtual_ranks=V)
    assert r.status == pb.CONVERGED
    assert_same(O, x, r, H, A)


# ------------------------------------------------------ plain fp64 dots ---
# the paper's non-reproducible comparison arm.

def test_plain_dots_mode(pb):
    A = gen.make_config("c1_2d64")
    S = solver(pb, A, history_capacity=600)
    b = gpu_b(pb, S, A)
    xe, re = S.solve(b, tol=1e-10, max_iter=500)
    He = S.history()
    xp, rp = S.solve(b, tol=1e-10, max_iter=500, dot_mode="plain")
    Hp = S.history()
    assert re.status == rp.status == pb.CONVERGED
    assert abs(rp.iterations - re.iterations) <= max(3, re.iterations // 10), (rp.iterations, re.iterations)
    assert rp.relres_true <= 1e-9
    # the same handle and launch geometry: deterministic
    xp2, rp2 = S.solve(b, tol=1e-10, max_iter=500, dot_mode="plain")
    assert np.array_equal(u64(S.history()), u64(Hp)) and np.array_equal(u64(xp2.cpu().numpy()), u64(xp.cpu().numpy()))
    # back to exact dots: the oracle's bits again
    xe2, re2 = S.solve(b, tol=1e-10, max_iter=500)
    assert np.array_equal(u64(S.history()), u64(He)) and np.array_equal(u64(xe2.cpu().numpy()), u64(xe.cpu().numpy()))
    O = oracle.PBiCGStab(A, tol=1e-10, max_iter=500)
    O.run()
    assert np.array_equal(u64(He), u64(O.history()))
    S.close()


def test_plain_dots_partition_witness(pb):
    # exact dots: identical bits for 1/2/4 ranks; plain dots: the grouping of
    # the fp64 sums follows the partition, so the trajectory does not
    import torch
    A = gen.stencil(3, 40, 100.0)
    hist = {}
    for mode in ("exact", "plain"):
        for V in (1, 2, 4):
            S = solver(pb, A, virtual_ranks=V, history_capacity=64)
            b = gpu_b(pb, S, A)
            S.start(b, tol=0.0, max_iter=40, dot_mode=mode)
            S.iterate(40)
            S.finish(None)
            hist[mode, V] = u64(S.history())
            S.close()
    assert all(np.array_equal(hist["exact", V], hist["exact", 1]) for V in (2, 4))
    assert any(not np.array_equal(hist["plain", V], hist["plain", 1]) for V in (2, 4))


# ------------------------------------------ Algorithm 1 with exact dots ---
# SURVEY §8(f) NEXT-1 second half: classic BiCGStab on the GPU, bit-exact
# against the oracle's orc_bicgstab_dots(exact = 1) (R-20).

def alg1_both(pb, A, tol, max_iter, **kw):
    S = solver(pb, A, history_capacity=max_iter + 2, **kw)
    b = gpu_b(pb, S, A)
    bh = b.cpu().numpy()
    st, it, xo, ho = oracle.bicgstab(A, bh, tol=tol, max_iter=max_iter, exact_dots=True)
    x, r = S.solve(b, tol=tol, max_iter=max_iter, method="bicgstab")
    H = S.history()
    S.close()
    return st, it, xo, ho, x.cpu().numpy(), r, H


@pytest.mark.parametrize("name", ["c1", "small3d", "rand", "dense"])
def test_alg1_matches_oracle(pb, name):
    A = {"c1": lambda: gen.make_config("c1_2d64"),
         "small3d": lambda: gen.stencil(3, 20, 100.0),
         "rand": lambda: gen.random_banded(20_000, seed=9, band=1500),
         "dense": lambda: gen.dense_as_sparse(57, seed=5, density=0.5)}[name]()
    st, it, xo, ho, x, r, H = alg1_both(pb, A, 1e-10, 3000)
    assert r.status == st and r.iterations == it, (r.status, st, r.iterations, it)
    assert np.array_equal(u64(H[:, oracle.H_RELRES]), u64(ho))
    assert np.array_equal(u64(x), u64(xo))
    if st == oracle.CONVERGED:
        assert r.relres_true <= 10 * 1e-10


def test_alg1_virtual_ranks_identical(pb):
    A = gen.stencil(3, 20, 100.0)
    ref = alg1_both(pb, A, 1e-10, 3000)
    for V in (2, 3):
        st, it, xo, ho, x, r, H = alg1_both(pb, A, 1e-10, 3000, virtual_ranks=V)
        assert np.array_equal(u64(x), u64(ref[4])) and np.array_equal(u64(H), u64(ref[6])), V


def test_alg1_q_convergence_and_errors(pb):
    # 1x1 diag(2): converges at the q check of the first iteration (x := x + a p)
    import torch
    A = gen.from_dense(np.array([[2.0]]))
    S = solver(pb, A)
    x, r = S.solve(torch.tensor([2.0], dtype=torch.float64, device="cuda"), method="bicgstab")
    assert r.status == pb.CONVERGED and r.iterations == 1 and x.item() == 1.0
    with pytest.raises(pb.PbcgError):
        S.solve(torch.tensor([2.0], dtype=torch.float64, device="cuda"), method="bicgstab", dot_mode="plain")
    S.close()
    st, it, xo, ho = oracle.bicgstab(A, np.array([2.0]), exact_dots=True)
    assert st == oracle.CONVERGED and it == 1 and xo[0] == 1.0


# ---------------------------------- residual replacement (NEXT-2, R-21) ---

@pytest.mark.parametrize("name,rr", [("c1", 10), ("small3d", 25), ("rand", 7)])
def test_residual_replacement_matches_oracle(pb, name, rr):
    A = {"c1": lambda: gen.make_config("c1_2d64"),
         "small3d": lambda: gen.stencil(3, 20, 100.0),
         "rand": lambda: gen.random_banded(20_000, seed=9, band=1500)}[name]()
    S = solver(pb, A, history_capacity=3001)
    b = gpu_b(pb, S, A)
    O = oracle.PBiCGStab(A, b=A.b if A.rhs == "given" else None, tol=1e-10, max_iter=3000, rr_period=rr)
    O.run()
    for poll, graphs in ((16, True), (7, True), (1, False)):
        x, r = S.solve(b, tol=1e-10, max_iter=3000, rr_period=rr, poll_every=poll, use_graphs=graphs)
        assert_same(O, x.cpu().numpy(), r, S.history(), A)
    assert O.replacements > 0
    S.close()


def test_residual_replacement_virtual_ranks(pb):
    A = gen.stencil(3, 20, 100.0)
    O = oracle.PBiCGStab(A, tol=1e-10, max_iter=3000, rr_period=13)
    O.run()
    S = solver(pb, A, history_capacity=3001, virtual_ranks=3)
    x, r = S.solve(gpu_b(pb, S, A), tol=1e-10, max_iter=3000, rr_period=13)
    assert_same(O, x.cpu().numpy(), r, S.history(), A)
    S.close()


# ------------------------------ right Jacobi preconditioning (NEXT-3, R-22) ---

@pytest.mark.parametrize("name", ["c1", "rand", "small3d"])
def test_jacobi_matches_oracle(pb, name):
    import torch
    A = {"c1": lambda: gen.make_config("c1_2d64"),
         "rand": lambda: gen.random_banded(20_000, seed=9, band=1500),
         "small3d": lambda: gen.stencil(3, 20, 100.0)}[name]()
    S0 = solver(pb, A)
    b = gpu_b(pb, S0, A)  # b of the original system
    S0.close()
    As, d = oracle.jacobi_right(A)
    O = oracle.PBiCGStab(As, b=b.cpu().numpy(), tol=1e-10, max_iter=3000)
    O.run()
    for V in (1, 3):
        S = solver(pb, A, history_capacity=3001, virtual_ranks=V, precond="jacobi")
        x, r = S.solve(b, tol=1e-10, max_iter=3000)
        assert r.iterations == O.iterations and r.status == O.status
        assert np.array_equal(u64(S.history()), u64(O.history()))
        assert np.array_equal(u64(S.vec("x")), u64(O.vec("x")))            # y
        assert np.array_equal(u64(x.cpu().numpy()), u64(O.vec("x") / d))  # x = D^-1 y
        S.close()


def test_jacobi_rejects_zero_diagonal(pb):
    A = gen.from_dense(np.array([[0.0, 1.0], [1.0, 2.0]]))
    with pytest.raises(pb.PbcgError) as e:
        solver(pb, A, precond="jacobi")
    assert e.value.rc == 1


# ------------------------------------------- 2x2 point-block Jacobi (R-23) ---

@pytest.mark.parametrize("name", ["c1", "rand", "small3d", "odd"])
def test_block_jacobi_matches_oracle(pb, name, monkeypatch):
    # B = A M^-1 formed on the GPU (pattern widened to whole column blocks,
    # M^-1 columns halo-exchanged) bit for bit as the oracle forms it; the
    # trajectory of B y = b, y (S.vec("x")) and x = M^-1 y; virtual ranks
    # with even first rows; fused small kernel and six-kernel path; the 1x1
    # tail block of an odd order
    import torch
    A = {"c1": lambda: gen.make_config("c1_2d64"),
         "rand": lambda: gen.random_banded(20_000, seed=9, band=1500),
         "small3d": lambda: gen.stencil(3, 20, 100.0),
         "odd": lambda: gen.random_banded(3_001, seed=5, band=300)}[name]()
    S0 = solver(pb, A)
    b = gpu_b(pb, S0, A)
    S0.close()
    B, M, Mi = oracle.block_jacobi_right(A)
    O = oracle.PBiCGStab(B, b=b.cpu().numpy(), tol=1e-10, max_iter=3000)
    O.run()
    assert O.status == oracle.CONVERGED
    want_x = u64(oracle.bj_apply(Mi, O.vec("x")))
    runs = [(1, "1"), (1, "0")] + ([(2, "1"), (4, "1")] if A.n % 8 == 0 else [])
    for V, small in runs:
        monkeypatch.setenv("PBCG_SMALL", small)
        S = solver(pb, A, history_capacity=3001, virtual_ranks=V, precond="bjacobi2")
        assert S.spmv_format()["nnz"] == B.nnz
        x, r = S.solve(b, tol=1e-10, max_iter=3000)
        assert r.iterations == O.iterations and r.status == O.status, (V, small)
        assert np.array_equal(u64(S.history()), u64(O.history())), (V, small)
        assert np.array_equal(u64(S.vec("x")), u64(O.vec("x")))  # y
        assert np.array_equal(u64(x.cpu().numpy()), want_x)      # x = M^-1 y
        S.close()


def test_block_jacobi_rejects(pb):
    # a singular 2x2 diagonal block; a rank whose first row is odd (3001 rows
    # on 2 virtual ranks: 0 | 1501)
    A = gen.from_dense(np.array([[1.0, 2.0, 0.0], [2.0, 4.0, 1.0], [0.0, 1.0, 3.0]]))
    with pytest.raises(pb.PbcgError) as e:
        solver(pb, A, precond="bjacobi2")
    assert e.value.rc == 1
    A = gen.random_banded(3_001, seed=5, band=300)
    assert pb.plan_partition(A.n, 2)[1] % 2 == 1
    with pytest.raises(pb.PbcgError) as e:
        solver(pb, A, precond="bjacobi2", virtual_ranks=2)
    assert e.value.rc == 1


# ----------------------------------------------- fused small-system kernel ---

@pytest.mark.parametrize("name", ["c1", "rand", "stencil3d", "ragged"])
def test_fused_small_kernel(pb, name, monkeypatch):
    # n <= 16384 rows, single rank, exact dots: one cooperative kernel runs
    # whole chunks of iterations (csrc/small.cuh).  Same bits as the
    # six-kernel path and as the oracle, resumed across launches of varied
    # length (the phase buffers alternate by iteration parity), sigma-sorted
    # rows (rand), a ragged last window (n % 256 != 0)
    import torch
    A = {"c1": lambda: gen.make_config("c1_2d64"),
         "rand": lambda: gen.random_banded(16_000, seed=9, band=1500),
         "stencil3d": lambda: gen.stencil(3, 25, 100.0),
         "ragged": lambda: gen.random_banded(3_001, seed=5, band=700)}[name]()
    M = 400
    got = {}
    for env in ("1", "0"):
        monkeypatch.setenv("PBCG_SMALL", env)
        S = solver(pb, A, history_capacity=M + 1)
        b = gpu_b(pb, S, A)
        S.start(b, tol=1e-10, max_iter=M)
        assert S.exec_mode() == int(env)
        for k in (1, 3, 7, 16, M):
            S.iterate(k)
        x = torch.zeros(A.n, dtype=torch.float64, device="cuda")
        r = S.finish(x)
        got[env] = (u64(x.cpu().numpy()), u64(S.history()), r.iterations, r.status)
        S.close()
    assert got["1"][2] == got["0"][2] and got["1"][3] == got["0"][3]
    assert np.array_equal(got["1"][0], got["0"][0]) and np.array_equal(got["1"][1], got["0"][1])
    monkeypatch.delenv("PBCG_SMALL")
    S, O, x, r, H = run_both(pb, A, tol=1e-10, max_iter=M)
    assert_same(O, x, r, H, A)


def test_fused_small_kernel_stops(pb):
    # max_iter inside a launch, and the modes that keep the six-kernel path
    import torch
    A = gen.make_config("c1_2d64")
    S, O, x, r, H = run_both(pb, A, tol=1e-30, max_iter=9)
    assert r.iterations == 9 and r.status == pb.MAXITER
    assert_same(O, x, r, H, A)
    S = solver(pb, A)
    b = gpu_b(pb, S, A)
    for kw, mode in ((dict(), 1), (dict(dot_mode="plain"), 1), (dict(method="bicgstab"), 0), (dict(rr_period=5), 0)):
        S.start(b, tol=1e-10, max_iter=20, **kw)
        assert S.exec_mode() == mode, kw
        S.iterate(3)
        S.finish(None)
    S.close()
    S = solver(pb, A, virtual_ranks=2)
    S.start(b, tol=1e-10, max_iter=20)
    assert S.exec_mode() == 0
    S.close()
    A = gen.stencil(3, 26, 100.0)  # 17,576 rows: above the threshold
    S = solver(pb, A)
    S.start(gpu_b(pb, S, A), tol=1e-10, max_iter=20)
    assert S.exec_mode() == 0
    S.close()


def test_fused_small_kernel_plain_dots(pb, monkeypatch):
    # plain fp64 dots in the fused kernel: per-thread fma chains, fixed warp
    # trees, partials summed in grid order -- deterministic for one grid,
    # converging like the exact solve; the six-kernel plain path groups the
    # sums differently (the non-reproducibility the paper describes)
    A = gen.make_config("c1_2d64")
    runs = {}
    for env in ("1", "1", "0"):
        monkeypatch.setenv("PBCG_SMALL", env)
        S = solver(pb, A, history_capacity=600)
        b = gpu_b(pb, S, A)
        x, r = S.solve(b, tol=1e-10, max_iter=500, dot_mode="plain")
        assert S.exec_mode() == int(env)
        assert r.status == pb.CONVERGED and r.relres_true <= 1e-9
        runs.setdefault(env, []).append((u64(x.cpu().numpy()), u64(S.history()), r.iterations))
        S.close()
    (x1, h1, i1), (x2, h2, i2) = runs["1"]
    assert i1 == i2 and np.array_equal(x1, x2) and np.array_equal(h1, h2)
    O = oracle.PBiCGStab(A, tol=1e-10, max_iter=500)
    O.run()
    assert abs(i1 - O.iterations) <= max(3, O.iterations // 10), (i1, O.iterations)


def test_solve_x0_zero_and_out_buffer(pb, monkeypatch):
    # x0=None starts from 0 on the device (pbcg_opts.x0_zero, no copy); out=
    # receives x (a pinned host tensor here): the same bits as x0 = zeros;
    # the polls overlap the next chunk, so the stop iteration is unchanged
    import torch
    A = gen.make_config("c1_2d64")
    S = solver(pb, A, history_capacity=600)
    b = gpu_b(pb, S, A)
    for small in ("1", "0"):
        monkeypatch.setenv("PBCG_SMALL", small)
        xa, ra = S.solve(b, x0=torch.zeros(A.n, dtype=torch.float64, device="cuda"), tol=1e-10, max_iter=500)
        Ha = S.history()
        bh = b.cpu().pin_memory()
        out = torch.empty(A.n, dtype=torch.float64).pin_memory()
        xb, rb = S.solve(bh, x0=None, out=out, tol=1e-10, max_iter=500, poll_every=7)
        assert xb.data_ptr() == out.data_ptr()
        assert ra.iterations == rb.iterations and ra.status == rb.status
        assert np.array_equal(u64(xa.cpu().numpy()), u64(out.numpy()))
        assert np.array_equal(u64(Ha), u64(S.history()))
        # a stop inside a chunk: max_iter not a multiple of poll_every
        xc, rc = S.solve(b, x0=None, tol=1e-30, max_iter=23, poll_every=16)
        assert rc.iterations == 23 and rc.status == pb.MAXITER
        # out= is written in place, never through a silent copy
        for bad in (torch.empty(A.n, dtype=torch.float32).pin_memory(), torch.empty(A.n + 1, dtype=torch.float64),
                    torch.empty(2 * A.n, dtype=torch.float64)[::2], torch.empty(A.n, dtype=torch.float64, device="cuda")):
            with pytest.raises(ValueError):
                S.solve(bh, x0=None, out=bad, tol=1e-10, max_iter=5)
    monkeypatch.delenv("PBCG_SMALL")
    O = oracle.PBiCGStab(A, tol=1e-10, max_iter=500)
    O.run()
    assert np.array_equal(u64(Ha), u64(O.history()))
    S.close()


@pytest.mark.parametrize("name", ["c1", "stencil3d"])
@pytest.mark.parametrize("dot_mode", ["exact", "plain"])
def test_fused_register_variant_same_bits(pb, name, dot_mode, monkeypatch):
    # the register-resident fused kernel (PBCG_SMALL_REG=1, the default where
    # it applies) and the shared-memory fused kernel give the same bits
    A = {"c1": lambda: gen.make_config("c1_2d64"), "stencil3d": lambda: gen.stencil(3, 24, 100.0)}[name]()
    got = {}
    for reg in ("1", "0"):
        monkeypatch.setenv("PBCG_SMALL_REG", reg)
        S = solver(pb, A, history_capacity=601)
        b = gpu_b(pb, S, A)
        x, r = S.solve(b, tol=1e-10, max_iter=600, dot_mode=dot_mode)
        assert S.exec_mode() == 1
        got[reg] = (u64(x.cpu().numpy()), u64(S.history()), r.iterations, r.status)
        S.close()
    assert got["1"][2:] == got["0"][2:]
    assert np.array_equal(got["1"][0], got["0"][0]) and np.array_equal(got["1"][1], got["0"][1])


# ---------------- pipelined 2x2 block Jacobi (R-25) ---

@pytest.mark.parametrize("name", ["c1", "rand", "small3d", "odd"])
def test_pipelined_block_jacobi_matches_oracle(pb, name):
    # M^-1 applied inside K2 (z_hat) and K3 (w_hat); the SpMVs run on A:
    # trajectory of A M^-1 y = b, y and x = M^-1 y bit for bit against the
    # oracle's op_apply, at 1 rank, 2/4 virtual ranks and the NCCL vehicle;
    # the odd order has a 1x1 tail block in the last rank's tail tile
    import torch
    A = {"c1": lambda: gen.make_config("c1_2d64"),
         "rand": lambda: gen.random_banded(20_000, seed=9, band=1500),
         "small3d": lambda: gen.stencil(3, 20, 100.0),
         "odd": lambda: gen.random_banded(3_001, seed=5, band=300)}[name]()
    S0 = solver(pb, A)
    b = gpu_b(pb, S0, A)
    S0.close()
    M, Mi = oracle.bj_blocks_c(A)
    O = oracle.PBiCGStab(A, b=b.cpu().numpy(), tol=1e-10, max_iter=3000, minv=Mi)
    O.run()
    assert O.status == oracle.CONVERGED
    want_x = u64(oracle.bj_apply(Mi, O.vec("x")))
    runs = [dict(), dict(force_nccl=True)] + ([dict(virtual_ranks=2), dict(virtual_ranks=4)] if A.n % 8 == 0 else [])
    for kw in runs:
        S = solver(pb, A, history_capacity=3001, precond="bjacobi2_pipe", **kw)
        assert S.spmv_format()["nnz"] == A.nnz  # A is stored as given
        x, r = S.solve(b, tol=1e-10, max_iter=3000)
        assert S.exec_mode() == 0
        assert r.iterations == O.iterations and r.status == O.status, kw
        assert np.array_equal(u64(S.history()), u64(O.history())), kw
        assert np.array_equal(u64(S.vec("x")), u64(O.vec("x"))), kw  # y
        assert np.array_equal(u64(x.cpu().numpy()), want_x), kw      # x = M^-1 y
        tr = oracle.true_relres(A, b.cpu().numpy(), oracle.bj_apply(Mi, O.vec("x")))[0]
        assert r.relres_true == tr, kw
        S.close()


def test_pipelined_block_jacobi_full_size_and_rejects(pb):
    # full C3 in the bench's launch configuration: first iterations bit-exact
    # (SELL-P SpMV on A, z_hat / w_hat from the stream kernels); Alg. 1 with
    # the pipelined preconditioner is EINVAL
    import torch
    A = gen.make_config("c3_3d128")
    M, Mi = oracle.bj_blocks_c(A)
    S = solver(pb, A, history_capacity=16, precond="bjacobi2_pipe")
    b = S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
    O = oracle.PBiCGStab(A, b=b.cpu().numpy(), tol=0.0, max_iter=8, minv=Mi)
    O.run(4)
    S.start(b, tol=0.0, max_iter=8)
    S.iterate(4)
    S.finish(None)
    assert np.array_equal(u64(S.history()), u64(O.history()))
    for k in ("z", "w", "t", "v", "x"):
        assert np.array_equal(u64(S.vec(k)), u64(O.vec(k))), k
    with pytest.raises(pb.PbcgError) as e:
        S.solve(b, method="bicgstab")
    assert e.value.rc == 1
    S.close()


@pytest.mark.parametrize("name", ["c1", "2d45", "3d15"])
def test_cluster_kernel_same_bits(pb, name, monkeypatch):
    # the one-cluster kernel (csrc/cluster.cuh: 16 CTAs, z/w over DSMEM,
    # barrier.cluster, dot words summed in CTA 0's shared memory) against the
    # register-resident fused kernel (PBCG_CLUSTER=0) and the oracle: same
    # bits, resumed across launches; plain dots deterministic and converging
    A = {"c1": lambda: gen.make_config("c1_2d64"), "2d45": lambda: gen.stencil(2, 45, 10.0),
         "3d15": lambda: gen.stencil(3, 15, 100.0)}[name]()
    got = {}
    for cl in ("1", "0"):
        monkeypatch.setenv("PBCG_CLUSTER", cl)
        S = solver(pb, A, history_capacity=601)
        b = gpu_b(pb, S, A)
        S.start(b, tol=1e-10, max_iter=600)
        assert S.exec_mode() == 1
        for k in (1, 3, 7, 600):
            S.iterate(k)
        x = torch_zeros(A.n)
        r = S.finish(x)
        got[cl] = (u64(x.cpu().numpy()), u64(S.history()), r.iterations, r.status)
        xp, rp = S.solve(b, tol=1e-10, max_iter=600, dot_mode="plain")
        xp2, rp2 = S.solve(b, tol=1e-10, max_iter=600, dot_mode="plain")
        assert rp.status == pb.CONVERGED and rp.iterations == rp2.iterations
        assert np.array_equal(u64(xp.cpu().numpy()), u64(xp2.cpu().numpy()))
        S.close()
    assert got["1"][2:] == got["0"][2:]
    assert np.array_equal(got["1"][0], got["0"][0]) and np.array_equal(got["1"][1], got["0"][1])
    O = oracle.PBiCGStab(A, tol=1e-10, max_iter=600)
    O.run()
    assert np.array_equal(got["1"][1], u64(O.history())) and np.array_equal(got["1"][0], u64(O.vec("x")))


def torch_zeros(n):
    import torch
    return torch.zeros(n, dtype=torch.float64, device="cuda")


@pytest.mark.parametrize("precond,method", [("none", "pbicgstab"), ("jacobi", "pbicgstab"), ("bjacobi2", "pbicgstab"),
                                            ("bjacobi2_pipe", "pbicgstab"), ("none", "bicgstab")])
def test_zero_start_chunked_same_bits(pb, precond, method):
    # x0 = 0 without reading x0 (pbcg_opts.x0_zero): r0 = b - A 0 = b bit for
    # bit, so start skips the residual SpMV; a pinned host b of >= 2^20 rows
    # is copied in chunks that overlap the scans and copies.  Same history and
    # x as an explicit x0 = +0 vector through the residual SpMV.
    import torch
    A = gen.stencil(2, 1024, 10.0)  # 2^20 rows: the chunked path
    S = solver(pb, A, history_capacity=64, precond=precond)
    b = gpu_b(pb, S, A)
    b[::1000] = -0.0  # signed zeros in b survive r0 = b - (+0)
    xa, ra = S.solve(b, x0=torch.zeros(A.n, dtype=torch.float64, device="cuda"), tol=0.0, max_iter=30, method=method)
    Ha = S.history()
    out = torch.empty(A.n, dtype=torch.float64).pin_memory()
    xb, rb = S.solve(b.cpu().pin_memory(), x0=None, out=out, tol=0.0, max_iter=30, method=method)
    assert ra.iterations == rb.iterations == 30 and ra.status == rb.status
    assert np.array_equal(u64(Ha), u64(S.history()))
    assert np.array_equal(u64(xa.cpu().numpy()), u64(out.numpy()))
    assert ra.relres_true == rb.relres_true
    S.close()


@pytest.mark.parametrize("scale", [2.0 ** -500, 2.0 ** 480])
def test_zero_start_full_range_init(pb, scale):
    # the x0 = 0 start's two-dot init kernel (PH_INIT0) corrects products
    # outside the fast zone like the four-dot init (R-24): a b scaled so that
    # (b,b) falls below 2^-960 (or reaches 2^960) gives the same history
    import torch
    A = gen.stencil(3, 40, 100.0)
    S = solver(pb, A, history_capacity=16)
    b = gpu_b(pb, S, A) * scale
    xa, ra = S.solve(b, x0=torch.zeros(A.n, dtype=torch.float64, device="cuda"), tol=0.0, max_iter=6)
    Ha = S.history()
    xb, rb = S.solve(b, x0=None, tol=0.0, max_iter=6)
    assert ra.status == rb.status and ra.iterations == rb.iterations
    assert np.array_equal(u64(Ha), u64(S.history()))
    assert np.array_equal(u64(xa.cpu().numpy()), u64(xb.cpu().numpy()))
    S.close()


@pytest.mark.parametrize("name", ["2d_ragged", "3d_ragged", "short_rows_wide_band", "sellv"])
def test_zero_start_chunk_plans(pb, name):
    # the chunked start on ragged sizes (chunk boundaries on 3,840-row unit
    # steps, a short last chunk), a 3D halo of 10,404 rows, and matrices the
    # plan rejects (a row reads beyond the next chunk; SELL-V): whole-copy
    # fallback.  Same history and x as the residual-SpMV path.
    import torch
    A = {"2d_ragged": lambda: gen.stencil(2, 1030, 10.0), "3d_ragged": lambda: gen.stencil(3, 102, 100.0),
         "short_rows_wide_band": lambda: gen.random_banded(1 << 20, lam=4.0, lmin=2, lmax=8, band=400_000),
         "sellv": lambda: gen.random_banded(1 << 20, lam=12.0, lmin=5, lmax=40, band=3000)}[name]()
    S = solver(pb, A, history_capacity=32)
    b = gpu_b(pb, S, A)
    xa, ra = S.solve(b, x0=torch.zeros(A.n, dtype=torch.float64, device="cuda"), tol=0.0, max_iter=12)
    Ha = S.history()
    out = torch.empty(A.n, dtype=torch.float64).pin_memory()
    xb, rb = S.solve(b.cpu().pin_memory(), x0=None, out=out, tol=0.0, max_iter=12)
    assert ra.iterations == rb.iterations == 12 and ra.status == rb.status and ra.digest == rb.digest
    assert np.array_equal(u64(Ha), u64(S.history()))
    assert np.array_equal(u64(xa.cpu().numpy()), u64(out.numpy()))
    S.close()
