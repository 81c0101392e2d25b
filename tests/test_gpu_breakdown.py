"""GPU parity of the in-loop stops of Algorithm 2:
BREAKDOWN_OMEGA / RHO / ALPHA and the mid-solve RANGE stops of phase A and
phase B, against the oracle pinned in tests/test_oracle_breakdown.py.

Defining passages: PAPER.md §2 Algorithm 2 l.76, l.81, l.82; SPEC.md l.231,
l.232, l.241; R-9, R-11, R-12, R-19.

Every case runs on four paths of the library: the six-kernel iteration
(K2 / SpMV / K3 stream kernels + side-stream finalize), the fused small-system
kernel (its register-resident and its shared-memory variants), three virtual
ranks, and the 1-rank NCCL vehicle.  Status, iteration count, the history rows
and x are compared bit for bit (for RANGE stops: the rows before the stop, the
values under the flag are not defined by R-9).
"""
import numpy as np
import pytest

import gen
import oracle
from a11_cases import EXACT, eps_for, range_case, tile

pytestmark = pytest.mark.gpu

PATHS = ["six_kernel", "fused", "fused_smem", "vranks3", "nccl"]


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def pb():
    import torch
    assert torch.cuda.is_available()
    import paper_2404_13216_b200 as pb
    return pb


def gpu_solve(pb, A, b, path, monkeypatch, **kw):
    import torch
    monkeypatch.setenv("PBCG_SMALL", "0" if path == "six_kernel" else "1")
    monkeypatch.setenv("PBCG_SMALL_REG", "0" if path == "fused_smem" else "1")
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=kw.get("max_iter", 100) + 1,
                  virtual_ranks=3 if path == "vranks3" else 1, force_nccl=(path == "nccl"))
    x, r = S.solve(torch.from_numpy(b).cuda(), **kw)
    want_mode = 1 if path in ("fused", "fused_smem") else 0
    assert S.exec_mode() == want_mode, (path, S.exec_mode())
    H = S.history()
    S.close()
    return x.cpu().numpy(), r, H


def _int_system(n, seed):
    rng = np.random.default_rng(seed)
    M = rng.integers(-3, 4, (n, n)).astype(float)
    M[np.arange(n), np.arange(n)] = np.abs(M).sum(1) + 2
    b = rng.integers(-5, 6, n).astype(float)
    if not b.any():
        b[0] = 1.0
    return M, b


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", sorted(EXACT))
def test_exact_zero_divisor(pb, name, path, monkeypatch):
    M, b0, outcome, iters = EXACT[name]
    A, b = tile(M, b0, 1000 if len(b0) != 4 else 750)  # 2,000-3,000 rows: many CTAs, ragged tails
    O = oracle.PBiCGStab(A, b=b, tol=1e-10, max_iter=50)
    O.run()
    assert oracle.STATUS_NAMES[O.status] == outcome and O.iterations == iters
    x, r, H = gpu_solve(pb, A, b, path, monkeypatch, tol=1e-10, max_iter=50)
    assert r.status == O.status and r.iterations == O.iterations, (path, r.status, r.iterations)
    assert np.array_equal(u64(H), u64(O.history())), path
    assert np.array_equal(u64(x), u64(O.vec("x"))), path


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("seed,kind,at", [(2, "rho", 1), (6, "rho", 1), (18, "alpha", 2)])
def test_relative_threshold(pb, seed, kind, at, path, monkeypatch):
    # breakdown_eps places the R-11 threshold just above |rho'| (or |d|) at
    # iteration `at`; 256 block-diagonal copies keep every ratio (the dots
    # scale by 2^8 exactly)
    M, b0 = _int_system(8, seed)
    eps = eps_for(M.tolist(), b0.tolist(), kind, at)
    A, b = tile(M, b0, 256)
    O = oracle.PBiCGStab(A, b=b, tol=0.0, eps=eps, max_iter=40)
    O.run()
    assert O.status == {"rho": oracle.BREAKDOWN_RHO, "alpha": oracle.BREAKDOWN_ALPHA}[kind]
    assert O.iterations == at + 1
    x, r, H = gpu_solve(pb, A, b, path, monkeypatch, tol=0.0, eps=eps, max_iter=40)
    assert r.status == O.status and r.iterations == O.iterations, (path, r.status, r.iterations)
    assert np.array_equal(u64(H), u64(O.history())), path
    assert np.array_equal(u64(x), u64(O.vec("x"))), path


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("phase", ["A", "B"])
def test_range_stop_mid_solve(pb, phase, path, monkeypatch):
    # range_mode "fast" (R-9): b * 2^-k: the first product below 2^-960 (R-9) falls in `phase` of an
    # iteration i >= 1; R-19 fixes the stop (A: before S6, iterations = i;
    # B: after S6, iterations = i + 1)
    A = gen.stencil(2, 50, 10.0)
    b = 1.0 + gen.uniform(A.n, 5, 0.0, 1.0)
    k, i, _, _ = range_case(oracle, A, b, phase)
    bs = b * 2.0 ** -k
    O = oracle.PBiCGStab(A, b=bs, tol=0.0, max_iter=80, range_mode="fast")
    O.run()
    assert O.status == oracle.RANGE and O.iterations == (i if phase == "A" else i + 1)
    x, r, H = gpu_solve(pb, A, bs, path, monkeypatch, tol=0.0, max_iter=80, range_mode="fast")
    assert r.status == pb.RANGE and r.iterations == O.iterations, (path, r.status, r.iterations)
    Ho = O.history()
    assert H.shape == Ho.shape
    assert np.array_equal(u64(H[: i + 1]), u64(Ho[: i + 1])), path  # rows before the stopped iteration
    if phase == "B":
        cols = [oracle.H_THETA, oracle.H_ETA, oracle.H_SIGMA, oracle.H_ZETA, oracle.H_OMEGA]
        assert np.array_equal(u64(H[i + 1, cols]), u64(Ho[i + 1, cols])), path
    assert np.array_equal(u64(x), u64(O.vec("x"))), path


# ---- full range (R-24): the default --------

def _full_case(name):
    """(A, b, tol, max_iter) systems whose dots leave the fast zone."""
    if name in ("under_a", "under_b"):  # b * 2^-k: products below 2^-960 from iteration i on (then subnormal dots)
        A = gen.stencil(2, 50, 10.0)
        b = 1.0 + gen.uniform(A.n, 5, 0.0, 1.0)
        k, i, _, _ = range_case(oracle, A, b, "A" if name == "under_a" else "B")
        return A, b * 2.0 ** -k, 0.0, 80
    if name == "under_converge":  # converges at the unscaled iteration, x scaled
        A = gen.stencil(2, 50, 10.0)
        return A, (1.0 + gen.uniform(A.n, 5, 0.0, 1.0)) * 2.0 ** -470, 1e-10, 400
    A = gen.stencil(3, 10, 100.0)  # b = A*1 * 2^k: products above 2^1000 (the FPE-overflow path)
    b = oracle.spmv(A, np.ones(A.n))
    return A, b * 2.0 ** (493 if name == "over_run" else 497), 0.0, 30


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("name", ["under_a", "under_b", "under_converge", "over_run", "over_stop"])
def test_full_range_solve(pb, name, path, monkeypatch):
    # the CTAs that meet products outside the fast zone correct them exactly
    # (K2/K3 stream kernels, init and true-residual multidots, fused kernels);
    # trajectories, outcome and x are the oracle's bit for bit.  over_stop:
    # a dot whose exact value overflows stops the solve with RANGE (R-24)
    A, b, tol, M = _full_case(name)
    O = oracle.PBiCGStab(A, b=b, tol=tol, max_iter=M)
    O.run()
    want = {"under_converge": oracle.CONVERGED, "over_stop": oracle.RANGE}.get(name, oracle.MAXITER)
    assert O.status == want, (name, O.status)
    Of = oracle.PBiCGStab(A, b=b, tol=tol, max_iter=M, range_mode="fast")
    Of.run()
    assert Of.status == oracle.RANGE and Of.iterations < O.iterations + (name == "over_stop")
    x, r, H = gpu_solve(pb, A, b, path, monkeypatch, tol=tol, max_iter=M)
    assert r.status == O.status and r.iterations == O.iterations, (path, r.status, r.iterations)
    Ho = O.history()
    if name == "over_stop":  # the row of the overflowing phase holds +-inf: compare the rows before it
        Ho, H = Ho[:-1], H[:-1]
    assert np.array_equal(u64(H), u64(Ho)), path
    assert np.array_equal(u64(x), u64(O.vec("x"))), path
    if name != "over_stop":
        tr = oracle.true_relres(A, b, O.vec("x"))[0]
        assert r.relres_true == tr or (np.isnan(tr) and np.isnan(r.relres_true))
