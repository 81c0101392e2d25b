"""Pins for the oracle's p-BiCGStab (§2 Algorithm 2) and plain
BiCGStab (Algorithm 1).

The oracle's floating-point Algorithm 2 is pinned to things it does not
compute itself:
* the textbook method: Algorithm 1 run in EXACT rational arithmetic gives the
  scalars the fp trajectory must track to rounding error (a transposed operand,
  wrong sign or index in any recurrence breaks this at the first iterations);
* the reading of Algorithm 2 (R-1..R-3) is itself pinned: Algorithm 2
  in exact rationals reproduces Algorithm 1's iterates exactly and terminates
  in <= n steps;
* definitional identities (S8/S4 products), auxiliary-vector
  invariants (w ~ Ar, s ~ Ap, z ~ As, y ~ Aq, r ~ b - Ax);
* closed forms (1x1 diag(2); a breakdown-at-init system);
* a dense direct solve (numpy.linalg.solve) on 100 random systems.
"""
import math
import struct
from fractions import Fraction as F

import numpy as np
import pytest

import gen
import oracle


def bits(v):
    return struct.unpack("<Q", struct.pack("<d", v))[0]


# ---------------------------------------------------------------- exact rational

def _mv(M, v):
    return [sum((M[i][j] * v[j] for j in range(len(v))), F(0)) for i in range(len(M))]


def _dot(a, b):
    return sum((x * y for x, y in zip(a, b)), F(0))


def alg1_exact(M, b, iters):
    """Algorithm 1 in exact rationals, x0 = 0."""
    n = len(b)
    x = [F(0)] * n
    r = list(b)
    r0 = list(r)
    p = list(r)
    out = []
    for _ in range(iters):
        s = _mv(M, p)
        a = _dot(r0, r) / _dot(r0, s)
        q = [ri - a * si for ri, si in zip(r, s)]
        y = _mv(M, q)
        yy = _dot(y, y)
        if yy == 0:
            x = [xi + a * pi for xi, pi in zip(x, p)]
            out.append(dict(alpha=a, omega=F(0), x=list(x), r=[F(0)] * n))
            break
        w = _dot(q, y) / yy
        x = [xi + a * pi + w * qi for xi, pi, qi in zip(x, p, q)]
        rn = [qi - w * yi for qi, yi in zip(q, y)]
        beta = (a / w) * _dot(r0, rn) / _dot(r0, r)
        out.append(dict(alpha=a, omega=w, x=list(x), r=list(rn), beta=beta))
        if all(v == 0 for v in rn):
            break
        p = [ri + beta * (pi - w * si) for ri, pi, si in zip(rn, p, s)]
        r = rn
    return out


def alg2_exact(M, b, iters):
    """Algorithm 2 in exact rationals, with readings
    R-1 (w0 := A r0), R-2 (scalar omega vs vector w), R-3 (i=0 copies)."""
    n = len(b)
    x = [F(0)] * n
    r = list(b)
    r0 = list(r)
    w = _mv(M, r)
    t = _mv(M, w)
    a = _dot(r0, r) / _dot(r0, w)
    out = []
    p = s = z = v = None
    beta = om = None
    for i in range(iters):
        if i == 0:
            p, s, z = list(r), list(w), list(t)
        else:
            p = [ri + beta * (pi - om * si) for ri, pi, si in zip(r, p, s)]
            s = [wi + beta * (si - om * zi) for wi, si, zi in zip(w, s, z)]
            z = [ti + beta * (zi - om * vi) for ti, zi, vi in zip(t, z, v)]
        q = [ri - a * si for ri, si in zip(r, s)]
        y = [wi - a * zi for wi, zi in zip(w, z)]
        v = _mv(M, z)
        yy = _dot(y, y)
        om = F(0) if yy == 0 else _dot(q, y) / yy
        x = [xi + a * pi + om * qi for xi, pi, qi in zip(x, p, q)]
        rn = [qi - om * yi for qi, yi in zip(q, y)]
        w = [yi - om * (ti - a * vi) for yi, ti, vi in zip(y, t, v)]
        t = _mv(M, w)
        out.append(dict(alpha=a, omega=om, x=list(x), r=list(rn)))
        if all(vv == 0 for vv in rn):
            break
        beta = (a / om) * _dot(r0, rn) / _dot(r0, r)
        a = _dot(r0, rn) / (_dot(r0, w) + beta * _dot(r0, s) - beta * om * _dot(r0, z))
        out[-1]["beta"] = beta
        r = rn
    return out


def _int_system(n, seed):
    rng = np.random.default_rng(seed)
    M = rng.integers(-3, 4, (n, n)).astype(float)
    M[np.arange(n), np.arange(n)] = np.abs(M).sum(1) + 2
    b = rng.integers(-5, 6, n).astype(float)
    if not b.any():
        b[0] = 1.0
    return M, b


def test_reading_alg2_equals_alg1_exactly():
    # pins readings R-1..R-3 (SURVEY.md App. A check): identical iterates,
    # exact zero residual after <= n steps
    for seed in range(3):
        M, b = _int_system(6, seed)
        Mf = [[F(v) for v in row] for row in M]
        bf = [F(v) for v in b]
        t1 = alg1_exact(Mf, bf, 10)
        t2 = alg2_exact(Mf, bf, 10)
        assert len(t1) == len(t2) <= 6
        for a1, a2 in zip(t1, t2):
            assert a1["alpha"] == a2["alpha"] and a1["omega"] == a2["omega"] and a1["x"] == a2["x"]
        assert all(v == 0 for v in t2[-1]["r"])
        xs = np.linalg.solve(M, b)
        assert np.allclose([float(v) for v in t2[-1]["x"]], xs, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("seed", range(4))
def test_fp_alg2_tracks_exact_alg1(seed):
    # the oracle's fp trajectory agrees with exact Algorithm 1 to rounding error
    n = 12
    M, b = _int_system(n, 100 + seed)
    A = gen.from_dense(M)
    S = oracle.PBiCGStab(A, b=b, tol=0.0, max_iter=4)
    S.run()
    H = S.history()
    ex = alg1_exact([[F(v) for v in row] for row in M], [F(v) for v in b], 4)
    # row 0 holds alpha_0 in H_ALPHA; row i+1 holds omega_i, and alpha_{i+1}
    assert math.isclose(H[0, oracle.H_ALPHA], float(ex[0]["alpha"]), rel_tol=1e-12)
    for i in range(3):
        assert math.isclose(H[i + 1, oracle.H_OMEGA], float(ex[i]["omega"]), rel_tol=1e-9), i
        assert math.isclose(H[i + 1, oracle.H_ALPHA], float(ex[i + 1]["alpha"]), rel_tol=1e-9), i
        assert math.isclose(H[i + 1, oracle.H_BETA], float(ex[i]["beta"]), rel_tol=1e-9), i
        rr = float(_dot(ex[i]["r"], ex[i]["r"]))
        assert math.isclose(H[i + 1, oracle.H_RR], rr, rel_tol=1e-8), i


def test_diag2_one_step():
    # SPEC.md l.243 / l.234: 1x1 diag(2), b=[2] -> converged in one step, x=[1]
    A = gen.from_dense(np.array([[2.0]]))
    S = oracle.PBiCGStab(A, b=[2.0], tol=1e-10, max_iter=10)
    S.run()
    assert S.status == oracle.CONVERGED and S.iterations == 1
    assert S.vec("x")[0] == 1.0
    assert S.history()[1, oracle.H_OMEGA] == 0.0  # (y,y) = 0 -> omega := 0 (R-12)


def test_i0_identities_and_definitional_products():
    # after i=0, s0 = A p0 and z0 = A s0 bitwise; v = A z and
    # t = A w are SpMV outputs by definition (S4, S8).
    M, b = _int_system(16, 7)
    A = gen.from_dense(M)
    S = oracle.PBiCGStab(A, b=b, tol=0.0, max_iter=1)
    S.step()
    p, s, z = S.vec("p"), S.vec("s"), S.vec("z")
    assert np.array_equal(s, oracle.spmv(A, p))
    assert np.array_equal(z, oracle.spmv(A, s))
    assert np.array_equal(S.vec("v"), oracle.spmv(A, z))
    assert np.array_equal(S.vec("t"), oracle.spmv(A, S.vec("w")))


def test_auxiliary_vector_invariants():
    # in exact arithmetic w = A r, s = A p, z = A s, y = A q, r = b - A x
    A = gen.stencil(2, 16, 10.0)
    S = oracle.PBiCGStab(A, tol=0.0, max_iter=8)
    S.run(8)
    v = {k: S.vec(k) for k in ("b", "x", "r", "p", "s", "z", "q", "y", "w")}
    Av = lambda u: oracle.spmv(A, u)
    nb = np.linalg.norm(v["b"])
    for lhs, rhs in [("w", Av(v["r"])), ("s", Av(v["p"])), ("z", Av(v["s"]))]:
        assert np.linalg.norm(v[lhs] - rhs) <= 1e-10 * nb, lhs
    assert np.linalg.norm(v["r"] - (v["b"] - Av(v["x"]))) <= 1e-10 * nb


def test_breakdown_init_closed_form():
    # A = [[0,1],[1,0]], b = [1,0]: r0 = b, w0 = A r0 = [0,1], (r0,w0) = 0
    A = gen.from_dense(np.array([[0.0, 1.0], [1.0, 0.0]]))
    S = oracle.PBiCGStab(A, b=[1.0, 0.0], tol=1e-10, max_iter=10)
    assert S.rc == 0 and S.status == oracle.BREAKDOWN_INIT and S.iterations == 0


def test_errors_and_degenerate():
    A = gen.from_dense(np.eye(3))
    assert oracle.PBiCGStab(A, b=[0.0, 0.0, 0.0]).rc == 1             # ||b|| = 0 -> EINVAL
    assert oracle.PBiCGStab(A, b=[1.0, math.nan, 0.0]).rc == 5        # NaN -> ENONFINITE
    B = gen.from_dense(np.array([[1.0, math.inf], [0.0, 1.0]]))
    assert oracle.PBiCGStab(B, b=[1.0, 1.0]).rc == 5
    S = oracle.PBiCGStab(A, b=[1.0, 2.0, 3.0], max_iter=0)
    assert S.status == oracle.MAXITER and S.iterations == 0
    S = oracle.PBiCGStab(A, b=[1.0, 2.0, 3.0], x0=[1.0, 2.0, 3.0])   # already solved
    assert S.status == oracle.CONVERGED and S.iterations == 0


def test_random_systems_vs_direct_solve():
    # 100 random well-conditioned systems of size 4-64 at
    # tol 1e-10, forward error <= 1e-6; l.380: true relres <= 10 tol
    rng = np.random.default_rng(2024)
    for k in range(100):
        n = int(rng.integers(4, 65))
        A = gen.dense_as_sparse(n, seed=k, density=0.5)
        M = np.zeros((n, n))
        for i in range(n):
            M[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
        b = rng.uniform(-1, 1, n)
        S = oracle.PBiCGStab(A, b=b, tol=1e-10, max_iter=1000)
        S.run()
        assert S.status == oracle.CONVERGED, (k, S.status)
        xs = np.linalg.solve(M, b)
        x = S.vec("x")
        assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)
        assert S.true_relres() <= 10 * 1e-10
        st, it, xb, _ = oracle.bicgstab(A, b, tol=1e-10, max_iter=1000)
        assert st == oracle.CONVERGED and np.linalg.norm(xb - xs) <= 1e-6 * np.linalg.norm(xs)


def test_c1_converges_and_matches_plain_bicgstab():
    # BASELINE.json configs[0]; north_star: final ||b-Ax||/||b|| agrees with a
    # plain-double BiCGStab within 1e-10
    A = gen.make_config("c1_2d64")
    S = oracle.PBiCGStab(A, tol=1e-10, max_iter=500)
    S.run()
    assert S.status == oracle.CONVERGED and 0 < S.iterations < 500
    H = S.history()
    assert H[-1, oracle.H_RELRES] <= 1e-10 < H[-2, oracle.H_RELRES]
    assert H[0, oracle.H_RELRES] == 1.0  # r0 = b (x0 = 0)
    tr = S.true_relres()
    b = S.vec("b")
    st, it, xb, _ = oracle.bicgstab(A, b, tol=1e-10, max_iter=500)
    assert st == oracle.CONVERGED
    tb = oracle.true_relres(A, b, xb)[0]
    assert abs(tr - tb) <= 1e-10
    assert np.abs(S.vec("x") - 1.0).max() < 1e-6  # b = A*ones


def test_deterministic():
    A = gen.stencil(2, 20, 10.0)
    S1 = oracle.PBiCGStab(A, tol=1e-10, max_iter=300)
    S2 = oracle.PBiCGStab(A, tol=1e-10, max_iter=300)
    S1.run(), S2.run()
    assert np.array_equal(S1.history().view(np.uint64), S2.history().view(np.uint64))
    assert np.array_equal(S1.vec("x").view(np.uint64), S2.vec("x").view(np.uint64))


# ---- Algorithm 1 with exact dots (the GPU's Alg. 1 arm) ----

def test_alg1_exact_dots_vs_direct_solve():
    # same pin as Alg. 2: random well-conditioned systems against a dense
    # direct solve, and the true residual within 10 tol
    rng = np.random.default_rng(77)
    for k in range(40):
        n = int(rng.integers(4, 65))
        A = gen.dense_as_sparse(n, seed=300 + k, density=0.5)
        M = np.zeros((n, n))
        for i in range(n):
            M[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
        b = rng.uniform(-1, 1, n)
        st, it, x, h = oracle.bicgstab(A, b, tol=1e-10, max_iter=1000, exact_dots=True)
        assert st == oracle.CONVERGED, (k, st)
        xs = np.linalg.solve(M, b)
        assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)
        assert oracle.true_relres(A, b, x)[0] <= 10 * 1e-10
        assert h[-1] <= 1e-10


def test_alg1_exact_vs_plain_dots_track():
    # the two dot choices differ by rounding only: on a well-conditioned
    # stencil the residual histories agree to many digits for the first
    # iterations and both reach the tolerance
    A = gen.stencil(2, 24, 10.0)
    b = oracle.spmv(A, np.ones(A.n))
    st0, it0, x0, h0 = oracle.bicgstab(A, b, tol=1e-10, max_iter=1000)
    st1, it1, x1, h1 = oracle.bicgstab(A, b, tol=1e-10, max_iter=1000, exact_dots=True)
    assert st0 == st1 == oracle.CONVERGED
    assert abs(it0 - it1) <= 3
    k = min(8, it0, it1)
    assert np.allclose(h0[:k], h1[:k], rtol=1e-9, atol=0)
    assert np.abs(x1 - 1.0).max() < 1e-6


def test_alg1_exact_dots_equals_alg2_solution():
    # Alg. 1 and Alg. 2 are the same method in exact arithmetic
    # (test_reading_alg2_equals_alg1_exactly); in fp both land on A^-1 b
    A = gen.make_config("c1_2d64")
    S = oracle.PBiCGStab(A, tol=1e-10, max_iter=500)
    S.run()
    st, it, x, h = oracle.bicgstab(A, S.vec("b"), tol=1e-10, max_iter=500, exact_dots=True)
    assert st == oracle.CONVERGED
    assert np.abs(x - S.vec("x")).max() < 1e-6
    assert abs(oracle.true_relres(A, S.vec("b"), x)[0] - S.true_relres()) <= 1e-10


# ---- residual replacement ----

def test_replacement_definitional_identities():
    # right after a replacement: r = b - A x, w = A r, s = A p, z = A s, t = A w, bitwise
    A = gen.stencil(2, 16, 10.0)
    S = oracle.PBiCGStab(A, tol=0.0, max_iter=50)
    S.run(7)
    S.replace()
    u = lambda a: np.ascontiguousarray(a).view(np.uint64)
    b, x = S.vec("b"), S.vec("x")
    assert np.array_equal(u(S.vec("r")), u(b - oracle.spmv(A, x)))
    assert np.array_equal(u(S.vec("w")), u(oracle.spmv(A, S.vec("r"))))
    assert np.array_equal(u(S.vec("s")), u(oracle.spmv(A, S.vec("p"))))
    assert np.array_equal(u(S.vec("z")), u(oracle.spmv(A, S.vec("s"))))
    assert np.array_equal(u(S.vec("t")), u(oracle.spmv(A, S.vec("w"))))
    assert S.replacements == 1


def test_replacement_period_semantics():
    A = gen.stencil(2, 20, 10.0)
    u = lambda a: np.ascontiguousarray(a).view(np.uint64)
    ref = oracle.PBiCGStab(A, tol=0.0, max_iter=40)
    ref.run()
    # a period beyond the run changes nothing
    S = oracle.PBiCGStab(A, tol=0.0, max_iter=40, rr_period=41)
    S.run()
    assert S.replacements == 0 and np.array_equal(u(S.history()), u(ref.history()))
    # period k: the first k iterations agree, replacements = floor(40 / k)
    S = oracle.PBiCGStab(A, tol=0.0, max_iter=40, rr_period=10)
    S.run()
    assert S.replacements == 3  # after iterations 10, 20, 30 (not after the last)
    assert np.array_equal(u(S.history()[:11]), u(ref.history()[:11]))


def test_replacement_converges_like_direct_solve():
    rng = np.random.default_rng(11)
    for k in range(20):
        n = int(rng.integers(8, 60))
        A = gen.dense_as_sparse(n, seed=500 + k, density=0.5)
        M = np.zeros((n, n))
        for i in range(n):
            M[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
        b = rng.uniform(-1, 1, n)
        S = oracle.PBiCGStab(A, b=b, tol=1e-10, max_iter=1000, rr_period=5)
        S.run()
        assert S.status == oracle.CONVERGED, (k, S.status)
        xs = np.linalg.solve(M, b)
        assert np.linalg.norm(S.vec("x") - xs) <= 1e-6 * np.linalg.norm(xs)
        assert S.true_relres() <= 10 * 1e-10


# ---- right Jacobi preconditioning (R-22) ----

def test_jacobi_right_scaling_identities():
    A = gen.random_banded(3000, seed=4, band=200)
    As, d = oracle.jacobi_right(A)
    # A' D = A column by column: the scaled diagonal is exactly 1
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    on = A.col == rows
    assert np.all(As.val[on] == 1.0)
    # one RN division per entry: |A'_ij d_j - A_ij| <= ulp/2 * |A_ij|
    back = As.val * d[A.col]
    assert np.all(np.abs(back - A.val) <= np.abs(A.val) * 2.0 ** -52)


def test_jacobi_preconditioned_solves():
    # converges to the direct solution of the ORIGINAL system (x = D^-1 y)
    rng = np.random.default_rng(21)
    for k in range(15):
        n = int(rng.integers(8, 60))
        A = gen.dense_as_sparse(n, seed=700 + k, density=0.5)
        M = np.zeros((n, n))
        for i in range(n):
            M[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
        b = rng.uniform(-1, 1, n)
        As, d = oracle.jacobi_right(A)
        S = oracle.PBiCGStab(As, b=b, tol=1e-10, max_iter=1000)
        S.run()
        assert S.status == oracle.CONVERGED, (k, S.status)
        x = S.vec("x") / d
        xs = np.linalg.solve(M, b)
        assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)


def test_jacobi_helps_a_badly_scaled_system():
    # rows scaled over 8 orders of magnitude: Jacobi restores the stencil's
    # convergence; the unpreconditioned solve needs more iterations
    A = gen.stencil(2, 24, 10.0)
    rng = np.random.default_rng(3)
    rs = 10.0 ** rng.uniform(-4, 4, A.n)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    B = gen.CSR(A.n, A.row_ptr, A.col, A.val * rs[rows])
    b = oracle.spmv(B, np.ones(B.n))
    S0 = oracle.PBiCGStab(B, b=b, tol=1e-10, max_iter=3000)
    S0.run()
    Bs, d = oracle.jacobi_right(B)
    S1 = oracle.PBiCGStab(Bs, b=b, tol=1e-10, max_iter=3000)
    S1.run()
    assert S1.status == oracle.CONVERGED
    assert S0.status != oracle.CONVERGED or S1.iterations < S0.iterations
    assert np.abs(S1.vec("x") / d - 1.0).max() < 1e-5


# ---- right 2x2 point-block Jacobi (R-23) ----

def test_oracle_fma_matches_libm():
    # the oracle's exact-rational fma against the C library's fma (glibc)
    import ctypes
    import ctypes.util
    libm = ctypes.CDLL(ctypes.util.find_library("m"))
    libm.fma.restype = ctypes.c_double
    libm.fma.argtypes = [ctypes.c_double] * 3
    rng = np.random.default_rng(5)
    vals = list(rng.uniform(-4, 4, 300) * 2.0 ** rng.integers(-1080, 1000, 300)) + \
        [0.0, -0.0, 1.0, -1.0, 2.0 ** -1074, -(2.0 ** -1074), 1.0 + 2.0 ** -52]
    for _ in range(3000):
        a, b, c = (vals[int(rng.integers(len(vals)))] for _ in range(3))
        want = libm.fma(a, b, c)
        got = oracle._fma(a, b, c)
        assert np.float64(got).view(np.uint64) == np.float64(want).view(np.uint64), (a, b, c, got, want)


def test_block_jacobi_identity_for_block_diagonal():
    # A block diagonal with exactly invertible blocks: B = A M^-1 is exactly
    # the identity (pattern widened to whole blocks), one iteration, x = M^-1 b
    blocks = [((2.0, 1.0), (0.0, 4.0)), ((1.0, -1.0), (1.0, 1.0)), ((8.0, 0.0), (0.0, 0.5))]
    n = 2 * len(blocks) + 1  # plus a 1x1 tail block
    D = np.zeros((n, n))
    for m, blk in enumerate(blocks):
        D[2 * m:2 * m + 2, 2 * m:2 * m + 2] = blk
    D[n - 1, n - 1] = 4.0
    A = gen.from_dense(D)
    B, M, Mi = oracle.block_jacobi_right(A)
    dense_b = np.zeros((n, n))
    for i in range(n):
        dense_b[i, B.col[B.row_ptr[i]:B.row_ptr[i + 1]]] = B.val[B.row_ptr[i]:B.row_ptr[i + 1]]
    assert np.array_equal(dense_b, np.eye(n))
    b = np.arange(1.0, n + 1.0)
    S = oracle.PBiCGStab(B, b=b, tol=1e-12, max_iter=5)
    S.run()
    assert S.status == oracle.CONVERGED and S.iterations == 1
    x = oracle.bj_apply(Mi, S.vec("x"))
    assert np.allclose(D @ x, b, rtol=0, atol=1e-14)


def test_block_jacobi_product_and_inverse():
    # B = A M^-1 entry by entry within a few ulps of the dense product, and
    # M^-1 within a few ulps of numpy's inverse of each block
    A = gen.random_banded(1001, seed=6, band=40)
    B, M, Mi = oracle.block_jacobi_right(A)
    for m in range(M.shape[0] - 1):
        blk = M[m].reshape(2, 2)
        assert np.allclose(Mi[m].reshape(2, 2), np.linalg.inv(blk), rtol=1e-14, atol=0)
    assert M.shape[0] == 501 and Mi[-1, 0] == 1.0 / M[-1, 0]  # 1x1 tail block (n odd)
    n = A.n
    Ad = np.zeros((n, n))
    for i in range(n):
        Ad[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
    Mid = np.zeros((n, n))
    for m in range(M.shape[0]):
        r0 = 2 * m
        if r0 + 1 < n:
            Mid[r0:r0 + 2, r0:r0 + 2] = Mi[m].reshape(2, 2)
        else:
            Mid[r0, r0] = Mi[m, 0]
    P = Ad @ Mid
    Bd = np.zeros((n, n))
    for i in range(n):
        Bd[i, B.col[B.row_ptr[i]:B.row_ptr[i + 1]]] = B.val[B.row_ptr[i]:B.row_ptr[i + 1]]
    assert np.all(np.abs(Bd - P) <= 4 * 2.0 ** -52 * (np.abs(Ad) @ np.abs(Mid)) + 1e-300)
    # the widened pattern holds every nonzero of the product
    assert np.all((P != 0) <= (Bd != 0) | (np.abs(P) < 1e-300))


def test_block_jacobi_preconditioned_solves():
    rng = np.random.default_rng(22)
    for k in range(12):
        n = int(rng.integers(8, 60))
        A = gen.dense_as_sparse(n, seed=800 + k, density=0.5)
        D = np.zeros((n, n))
        for i in range(n):
            D[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
        b = rng.uniform(-1, 1, n)
        B, M, Mi = oracle.block_jacobi_right(A)
        S = oracle.PBiCGStab(B, b=b, tol=1e-10, max_iter=1000)
        S.run()
        assert S.status == oracle.CONVERGED, (k, S.status)
        x = oracle.bj_apply(Mi, S.vec("x"))
        xs = np.linalg.solve(D, b)
        assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)
        # y0 = M x0 then x = M^-1 y round trip
        y = oracle.bj_apply(M, xs)
        assert np.allclose(oracle.bj_apply(Mi, y), xs, rtol=1e-13, atol=1e-15)


# ---- pipelined right 2x2 block Jacobi (R-25) ----
# Algorithm 2 on B = A M^-1 where every product B u is evaluated inside the
# iteration as A (M^-1 u): u_hat = M^-1 u (orc_bj_apply), then A's fma chain.

def _dense(A):
    D = np.zeros((A.n, A.n))
    for i in range(A.n):
        D[i, A.col[A.row_ptr[i]:A.row_ptr[i + 1]]] = A.val[A.row_ptr[i]:A.row_ptr[i + 1]]
    return D


def test_bj_apply_c_twin():
    # the C block apply inside the oracle's operator == the Python one (pinned
    # against libm fma), incl. odd order and signed zeros
    rng = np.random.default_rng(5)
    for n in (1, 2, 7, 64, 1001):
        Q = rng.normal(size=((n + 1) // 2, 4))
        x = rng.normal(size=n)
        x[rng.random(n) < 0.1] = -0.0
        Q[rng.random(Q.shape) < 0.1] = 0.0
        assert np.array_equal(oracle.bj_apply_c(Q, x).view(np.uint64), oracle.bj_apply(Q, x).view(np.uint64))


def test_bj_blocks_c_twin():
    # the C blocks (full-size tests) == block_jacobi_right's, bit for bit
    for A in (gen.random_banded(1001, seed=6, band=40), gen.stencil(2, 13, 10.0), gen.dense_as_sparse(9, seed=2)):
        B, M, Mi = oracle.block_jacobi_right(A)
        M2, Mi2 = oracle.bj_blocks_c(A)
        assert np.array_equal(M.view(np.uint64), M2.view(np.uint64))
        assert np.array_equal(Mi.view(np.uint64), Mi2.view(np.uint64))
    with pytest.raises(ValueError):
        oracle.bj_blocks_c(gen.from_dense(np.array([[1.0, 2.0], [2.0, 4.0]])))


def test_pipelined_bjacobi_operator_products():
    # after one step: s = B p, z = B s, v = B z, t = B w with B u := spmv(A, bj_apply(M^-1, u))
    # -- the composition of two pinned routines, right (not left) of A
    A = gen.random_banded(300, seed=4, band=20)
    B, M, Mi = oracle.block_jacobi_right(A)
    S = oracle.PBiCGStab(A, b=A.b, tol=0.0, max_iter=3, minv=Mi)
    S.step()
    Bop = lambda u: oracle.spmv(A, oracle.bj_apply(Mi, u))
    u = lambda a: a.view(np.uint64)
    assert np.array_equal(u(S.vec("s")), u(Bop(S.vec("p"))))
    assert np.array_equal(u(S.vec("z")), u(Bop(S.vec("s"))))
    assert np.array_equal(u(S.vec("v")), u(Bop(S.vec("z"))))
    assert np.array_equal(u(S.vec("t")), u(Bop(S.vec("w"))))
    assert not np.array_equal(u(S.vec("z")), u(oracle.bj_apply(Mi, oracle.spmv(A, S.vec("s")))))  # not M^-1 A


@pytest.mark.parametrize("seed", range(3))
def test_pipelined_bjacobi_tracks_exact(seed):
    # exact-rational Algorithm 2 on the matrix A M^-1 (M^-1 = the oracle's
    # rounded blocks): the fp trajectory agrees to rounding error
    from a11_cases import alg2_exact
    n = 10
    M0, b = _int_system(n, 300 + seed)
    A = gen.from_dense(M0)
    B, M, Mi = oracle.block_jacobi_right(A)
    Mid = np.zeros((n, n))
    for m in range(Mi.shape[0]):
        Mid[2 * m:2 * m + 2, 2 * m:2 * m + 2] = Mi[m].reshape(2, 2)
    P = [[sum(F(M0[i][k]) * F(Mid[k][j]) for k in range(n)) for j in range(n)] for i in range(n)]
    ex = alg2_exact(P, [F(v) for v in b], 4)
    S = oracle.PBiCGStab(A, b=b, tol=0.0, max_iter=4, minv=Mi)
    S.run()
    H = S.history()
    for i in range(3):
        assert math.isclose(H[i + 1, oracle.H_OMEGA], float(ex[i]["omega"]), rel_tol=1e-9), i
        assert math.isclose(H[i, oracle.H_ALPHA], float(ex[i]["alpha"]), rel_tol=1e-9), i
        assert math.isclose(H[i + 1, oracle.H_RR], float(ex[i]["rr"]), rel_tol=1e-8), i


def test_pipelined_bjacobi_solves():
    rng = np.random.default_rng(23)
    for k in range(12):
        n = int(rng.integers(8, 60))
        A = gen.dense_as_sparse(n, seed=900 + k, density=0.5)
        D = _dense(A)
        b = rng.uniform(-1, 1, n)
        B, M, Mi = oracle.block_jacobi_right(A)
        S = oracle.PBiCGStab(A, b=b, tol=1e-10, max_iter=1000, minv=Mi)
        S.run()
        assert S.status == oracle.CONVERGED, (k, S.status)
        x = oracle.bj_apply(Mi, S.vec("x"))
        xs = np.linalg.solve(D, b)
        assert np.linalg.norm(x - xs) <= 1e-6 * np.linalg.norm(xs)
        assert oracle.true_relres(A, b, x)[0] <= 10 * 1e-10
        # the stored-B arm (R-23) solves the same system; different roundings
        S2 = oracle.PBiCGStab(B, b=b, tol=1e-10, max_iter=1000)
        S2.run()
        assert np.linalg.norm(oracle.bj_apply(Mi, S2.vec("x")) - x) <= 1e-6 * np.linalg.norm(xs)


def test_pipelined_bjacobi_block_diagonal():
    # M = A's blocks: A (M^-1 u) = u up to rounding -> converges in <= 2 iterations
    rng = np.random.default_rng(8)
    n = 41
    D = np.zeros((n, n))
    for m in range(n // 2):
        D[2 * m:2 * m + 2, 2 * m:2 * m + 2] = rng.uniform(1, 2, (2, 2)) + 3 * np.eye(2)
    D[n - 1, n - 1] = 3.0
    A = gen.from_dense(D)
    B, M, Mi = oracle.block_jacobi_right(A)
    b = rng.uniform(-1, 1, n)
    S = oracle.PBiCGStab(A, b=b, tol=1e-12, max_iter=10, minv=Mi)
    S.run()
    assert S.status == oracle.CONVERGED and S.iterations <= 2
    assert np.allclose(D @ oracle.bj_apply(Mi, S.vec("x")), b, rtol=0, atol=1e-12)
