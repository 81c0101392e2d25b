"""Pins for the oracle's in-loop stops of Algorithm 2:
BREAKDOWN_OMEGA, BREAKDOWN_RHO, BREAKDOWN_ALPHA and the mid-solve RANGE stops.

Defining passages: PAPER.md §2 Algorithm 2 l.76 (omega = (q,y)/(y,y)),
l.81 (beta, divisor rho = (r0, r_i)), l.82 (alpha' = (r0,r')/d)
(omega := 0 when (y,y) = 0), l.232 (rho breakdown, relative threshold),
l.241 (alpha-denominator breakdown); readings R-9, R-11, R-12, R-19.

Nothing here re-types the oracle: the expected outcomes come from
* exact rational arithmetic (tests/a11_cases.alg2_exact) on systems where
  binary64 with FMA policy F is exact, so the oracle must reproduce the exact
  trajectory bit for bit and stop where the exact divisor is zero;
* Cauchy-Schwarz and exact ratios |rho'|/(NORM(r^) NORM(r')) that place the
  relative threshold of R-11 on either side of |rho'| (or |d|);
* exact power-of-two scaling: with b * 2^-k every vector scales by 2^-k and
  every dot by 2^-2k, so the first product below 2^-960 (R-9) -- and hence
  the phase and iteration of the RANGE stop (R-19) -- is read off the
  unscaled run's vectors by numpy.
A wrong order of the S10 checks, a wrong threshold formula, a sign or
operand error in d, or a RANGE stop on the wrong side of S6 fails one of them.
"""
import math

import numpy as np
import pytest

import gen
import oracle
from a11_cases import EXACT, alg2_exact, eps_for, is_short_dyadic, range_case, tile

STATUS = {"breakdown_omega": oracle.BREAKDOWN_OMEGA, "breakdown_rho": oracle.BREAKDOWN_RHO,
          "breakdown_alpha": oracle.BREAKDOWN_ALPHA}


def u64(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


@pytest.mark.parametrize("name", sorted(EXACT))
def test_exact_zero_divisor_closed_form(name):
    M, b, outcome, iters = EXACT[name]
    tr = alg2_exact(M, b, 10)
    # the closed form: exact dyadic trajectory, stop at the expected divisor
    for e in tr:
        for key in ("alpha", "omega", "rho1", "rr"):
            assert is_short_dyadic(e[key]), (name, key)
        assert all(is_short_dyadic(c) for c in e["x"] + e["r"])
    last = tr[-1]
    assert len(tr) == iters
    assert any(c != 0 for c in last["r"])  # not converged
    if outcome == "breakdown_omega":
        assert last["omega"] == 0
        assert last["rho1"] == 0  # (r^, q) = 0 exactly: only the check order decides (R-11/R-12)
    elif outcome == "breakdown_rho":
        assert last["omega"] != 0 and last["rho1"] == 0
    else:
        assert last["omega"] != 0 and last["rho1"] != 0 and last["d"] == 0
    for m in (1, 7):
        A, bb = tile(M, b, m)
        O = oracle.PBiCGStab(A, b=bb, tol=1e-10, max_iter=50)
        O.run()
        assert O.status == STATUS[outcome] and O.iterations == iters, (name, m, O.status, O.iterations)
        H = O.history()
        for i, e in enumerate(tr):
            assert H[i + 1, oracle.H_OMEGA] == float(e["omega"])
            assert H[i + 1, oracle.H_RHO] == m * float(e["rho1"])
            assert H[i + 1, oracle.H_RR] == m * float(e["rr"])
            assert H[i, oracle.H_ALPHA] == float(e["alpha"])
        assert np.array_equal(O.vec("x"), np.tile([float(c) for c in last["x"]], m))
        assert np.array_equal(O.vec("r"), np.tile([float(c) for c in last["r"]], m))


def _int_system(n, seed):
    rng = np.random.default_rng(seed)
    M = rng.integers(-3, 4, (n, n)).astype(float)
    M[np.arange(n), np.arange(n)] = np.abs(M).sum(1) + 2
    b = rng.integers(-5, 6, n).astype(float)
    if not b.any():
        b[0] = 1.0
    return M, b


# (seed, kind, at): eps_for finds a threshold window for these (8x8 systems)
THRESHOLD_CASES = [(0, "rho", 0), (2, "rho", 1), (2, "rho", 2), (6, "rho", 1), (18, "alpha", 2)]


@pytest.mark.parametrize("seed,kind,at", THRESHOLD_CASES)
def test_relative_threshold_sides(seed, kind, at):
    # R-11: thr = max(RN(RN(eps NORM(r^)) sqrt(rr)), 1e-300).  eps just above
    # the exact ratio |rho'| / (NORM(r^) NORM(r')) (resp. |d| / ...) stops the
    # solve at that iteration with that outcome; just below, it does not.
    M, b = _int_system(8, seed)
    eps = eps_for(M.tolist(), b.tolist(), kind, at)
    assert eps is not None
    A = gen.from_dense(M)
    O = oracle.PBiCGStab(A, b=b, tol=0.0, eps=eps, max_iter=40)
    O.run()
    assert O.status == STATUS["breakdown_" + kind] and O.iterations == at + 1, (O.status, O.iterations)
    O2 = oracle.PBiCGStab(A, b=b, tol=0.0, eps=eps * (1 - 1e-4), max_iter=40)
    O2.run()
    assert not (O2.status == O.status and O2.iterations == at + 1)
    # the history up to the stop is the unstopped run's (the check only decides)
    O3 = oracle.PBiCGStab(A, b=b, tol=0.0, max_iter=at + 1)
    O3.run()
    H, H3 = O.history(), O3.history()
    cols = [oracle.H_THETA, oracle.H_ETA, oracle.H_SIGMA, oracle.H_ZETA, oracle.H_OMEGA, oracle.H_RHO,
            oracle.H_DELTA, oracle.H_RR, oracle.H_RELRES]
    assert np.array_equal(u64(H[:, cols]), u64(H3[:, cols]))
    assert np.array_equal(u64(O.vec("x")), u64(O3.vec("x")))


def test_cauchy_schwarz_eps_one():
    # eps = 1.01: |rho'| <= NORM(r^) NORM(r') < thr for any system, so every
    # solve that neither converges nor hits omega = 0 stops after ONE
    # iteration with BREAKDOWN_RHO
    for seed in range(6):
        M, b = _int_system(10, 40 + seed)
        O = oracle.PBiCGStab(gen.from_dense(M), b=b, tol=0.0, eps=1.01, max_iter=40)
        O.run()
        assert O.status == oracle.BREAKDOWN_RHO and O.iterations == 1


@pytest.mark.parametrize("phase", ["A", "B"])
def test_range_stop_mid_solve(phase):
    # range_mode "fast" -- R-9 / R-19: b * 2^-k; the first product below 2^-960 falls in `phase`
    # of iteration i >= 1.  Phase A: stop before S6 (x unchanged, iterations
    # = i).  Phase B: stop after S6 (iterations = i + 1).  Every history row
    # before the stop is the unscaled row with the dots times 2^-2k.
    A = gen.stencil(2, 12, 10.0)
    b = 1.0 + gen.uniform(A.n, 5, 0.0, 1.0)
    case = range_case(oracle, A, b, phase)
    assert case is not None
    k, i, H, xs = case
    O = oracle.PBiCGStab(A, b=b * 2.0 ** -k, tol=0.0, max_iter=60, range_mode="fast")
    O.run()
    want_it = i if phase == "A" else i + 1
    assert O.status == oracle.RANGE and O.iterations == want_it, (k, i, O.status, O.iterations)
    Hs = O.history()
    dots = [oracle.H_THETA, oracle.H_ETA, oracle.H_SIGMA, oracle.H_ZETA, oracle.H_RHO, oracle.H_DELTA, oracle.H_RR]
    same = [oracle.H_OMEGA, oracle.H_RELRES, oracle.H_BETA, oracle.H_ALPHA]
    rows = slice(0, i + 1)  # rows 0..i: init and iterations 0..i-1 (all unflagged)
    assert np.array_equal(u64(Hs[rows][:, dots]), u64(H[rows][:, dots] * 2.0 ** (-2 * k)))
    assert np.array_equal(u64(Hs[rows][:, same]), u64(H[rows][:, same]))
    if phase == "B":  # the phase-A columns of the stopped iteration were unflagged
        a_cols = [oracle.H_THETA, oracle.H_ETA, oracle.H_SIGMA, oracle.H_ZETA]
        assert np.array_equal(u64(Hs[i + 1, a_cols]), u64(H[i + 1, a_cols] * 2.0 ** (-2 * k)))
        assert Hs[i + 1, oracle.H_OMEGA] == H[i + 1, oracle.H_OMEGA]
    assert np.array_equal(u64(O.vec("x")), u64(xs[want_it] * 2.0 ** -k))


# ---- full range (R-24): dots exact over the
# whole binary64 range, so a product outside the fast
# zone no longer stops the solve ----

DOTS = [oracle.H_THETA, oracle.H_ETA, oracle.H_SIGMA, oracle.H_ZETA, oracle.H_RHO, oracle.H_DELTA, oracle.H_RR]
SAME = [oracle.H_OMEGA, oracle.H_RELRES, oracle.H_BETA, oracle.H_ALPHA]


@pytest.mark.parametrize("phase", ["A", "B"])
def test_full_range_continues_past_the_fast_zone(phase):
    # the systems of test_range_stop_mid_solve: with full range the solve runs
    # on, and every row is the unscaled row (dots times 2^-2k) as long as the
    # scaled dots stay normal binary64 numbers (exact power-of-two scaling)
    A = gen.stencil(2, 12, 10.0)
    b = 1.0 + gen.uniform(A.n, 5, 0.0, 1.0)
    k, i, _, _ = range_case(oracle, A, b, phase)
    M = 60
    O0 = oracle.PBiCGStab(A, b=b, tol=0.0, max_iter=M)
    O0.run()
    H0 = O0.history()
    O = oracle.PBiCGStab(A, b=b * 2.0 ** -k, tol=0.0, max_iter=M)
    O.run()
    H = O.history()
    scaled = H0[:, DOTS] * 2.0 ** (-2 * k)
    small = np.any((scaled != 0) & (np.abs(scaled) < 2.0 ** -1022), axis=1)
    last = int(np.argmax(small)) if small.any() else H0.shape[0]  # first row with a subnormal dot
    assert last > i + 2, (last, i)
    assert np.array_equal(u64(H[:last, DOTS]), u64(scaled[:last]))
    assert np.array_equal(u64(H[:last, SAME]), u64(H0[:last, SAME]))
    if last == H0.shape[0]:
        assert O.status == oracle.MAXITER and np.array_equal(u64(O.vec("x")), u64(O0.vec("x") * 2.0 ** -k))


def test_full_range_converges_bit_exact_scaled():
    # tol 1e-10: the scaled system converges in the same iteration with
    # x = x_unscaled * 2^-k, although its products leave the fast zone
    A = gen.stencil(2, 12, 10.0)
    b = 1.0 + gen.uniform(A.n, 5, 0.0, 1.0)
    O0 = oracle.PBiCGStab(A, b=b, tol=1e-10, max_iter=300)
    O0.run()
    assert O0.status == oracle.CONVERGED
    for k in (440, 470):
        Of = oracle.PBiCGStab(A, b=b * 2.0 ** -k, tol=1e-10, max_iter=300, range_mode="fast")
        Of.run()
        assert Of.status == oracle.RANGE
        O = oracle.PBiCGStab(A, b=b * 2.0 ** -k, tol=1e-10, max_iter=300)
        O.run()
        assert O.status == oracle.CONVERGED and O.iterations == O0.iterations, k
        assert np.array_equal(u64(O.vec("x")), u64(O0.vec("x") * 2.0 ** -k))
        assert np.array_equal(u64(O.history()[:, SAME]), u64(O0.history()[:, SAME]))


def _overflow_system(name):
    if name == "2d":
        A = gen.stencil(2, 12, 10.0)
        return A, 1.0 + gen.uniform(A.n, 5, 0.0, 1.0)
    A = gen.stencil(3, 10, 100.0)  # b = A*1: the residual climbs ~2^12 before it falls
    return A, oracle.spmv(A, np.ones(A.n))


@pytest.mark.parametrize("name,k", [("2d", 501), ("2d", 503), ("2d", 506), ("3d", 493), ("3d", 497)])
def test_full_range_overflow_zone(name, k):
    # b * 2^+k: products above 2^1000 (outside the fast zone: "fast" stops at
    # init) are exact with full range; the solve stops with RANGE exactly at
    # the first dot whose exact value rounds to +-inf (|dot| 2^2k >= 2^1024),
    # (phase A of iteration i stops with iterations = i, R-19)
    A, b = _overflow_system(name)
    M = 30
    O0 = oracle.PBiCGStab(A, b=b, tol=0.0, max_iter=M)
    O0.run()
    H0 = O0.history()
    Of = oracle.PBiCGStab(A, b=b * 2.0 ** k, tol=0.0, max_iter=M, range_mode="fast")
    Of.run()
    assert Of.status == oracle.RANGE
    # the first phase (init, then A and B of each iteration) with an overflowing dot
    rows = []
    rows.append(("I", 0, [oracle.H_RHO, oracle.H_DELTA, oracle.H_RR]))
    for r in range(1, H0.shape[0]):
        rows.append(("A", r, [oracle.H_THETA, oracle.H_ETA, oracle.H_SIGMA, oracle.H_ZETA]))
        rows.append(("B", r, [oracle.H_RHO, oracle.H_DELTA, oracle.H_RR]))
    lim = 1024 - 2 * k
    stop = next(((ph, r) for ph, r, cols in rows if np.log2(np.abs(H0[r, cols]).max()) >= lim), None)
    assert stop is None or all(abs(np.log2(np.abs(H0[r, c]).max()) - lim) > 1e-9 for _, r, c in rows)
    O = oracle.PBiCGStab(A, b=b * 2.0 ** k, tol=0.0, max_iter=M)
    O.run()
    if stop is None:
        assert O.status == oracle.MAXITER and O.iterations == M
        good = H0.shape[0]
    else:
        ph, r = stop
        assert O.status == oracle.RANGE
        assert O.iterations == {"I": 0, "A": r - 1, "B": r}[ph], (stop, O.iterations)
        good = r if ph != "I" else 0
    H = O.history()
    assert np.array_equal(u64(H[:good, DOTS]), u64(H0[:good, DOTS] * 2.0 ** (2 * k)))
    assert np.array_equal(u64(H[:good, SAME]), u64(H0[:good, SAME]))
