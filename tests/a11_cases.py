"""Systems whose in-loop stop of Algorithm 2 is known in closed form (SURVEY
§8(a) row a11; readings R-11, R-12, R-19).

Test infrastructure shared by tests/test_oracle_solver.py (CPU pins of the
oracle) and tests/test_gpu_breakdown.py (GPU parity).  Nothing here calls the
CUDA library; the exact-rational evaluation below never calls the oracle.

* EXACT: small integer systems on which Algorithm 2 runs in exact dyadic
  arithmetic -- every vector entry and scalar of the first iterations is a
  short dyadic rational, so binary64 with FMA policy F computes them without
  rounding -- and a divisor of PAPER.md l.76 / l.81 / l.82 is exactly zero:
    omega_i = (q,y)/(y,y) = 0 with r' != 0 (l.76, R-12),
    rho' = (r^, r_{i+1}) = 0 with r' != 0 (l.81),
    d = (r^, w') + beta (r^, s) - beta omega (r^, z) = 0 (l.82).
  Found by a brute-force search over 2x2..4x4 matrices with entries in
  [-2, 2]; `alg2_exact` re-derives every expectation.
* `tile`: m block-diagonal copies (all dots scale by m exactly, the scalars
  do not change), so the same closed form holds at sizes that span many CTAs
  and several ranks.
* `eps_for`: a breakdown_eps that puts the relative threshold
  thr = eps NORM(r^) NORM(r') (R-11) just above |rho'| (or |d|) at a chosen
  iteration and below every earlier one -- from exact rationals.
* `range_case`: b scaled by 2^-k.  Every vector scales by 2^-k and every dot
  by 2^-2k exactly, the scalars are unchanged, so the first product below
  2^-960 (R-9) -- phase A or phase B, R-19 -- is predicted from the unscaled
  run's vectors with numpy.
"""
from __future__ import annotations

import math
from fractions import Fraction as F

import numpy as np

import gen

# name -> (matrix rows, b, outcome, iterations, first iteration index i of the stop)
EXACT = {
    # PAPER.md l.76 with (q, y) = 0 at i = 1: omega_1 = 0, r_2 = q_1 != 0.
    # Because (r^, q_i) = 0 in exact arithmetic, rho' = 0 too: the order
    # "omega = 0 before |rho'| <= thr" (R-11, R-12) decides the outcome.
    "omega_i1": ([[-1, 0, -2], [1, 0, 0], [0, -2, 2]], [-2, 2, 0], "breakdown_omega", 2),
    # singular: A = [[1,1],[0,0]], b = (1,1): alpha0 = 1, y = w0 - t0 = 0, q = (-1, 1)
    "omega_i0": ([[1, 1], [0, 0]], [1, 1], "breakdown_omega", 1),
    # (r^, r_2) = 0 at i = 1 with omega_1 != 0
    "rho_i1": ([[1, 1, 0, 1], [1, -2, -2, 0], [-1, 2, 2, 1], [0, 2, 1, 1]], [0, 0, 0, -2], "breakdown_rho", 2),
    "rho_i0": ([[2, -1, -2], [0, 2, 0], [1, -1, 0]], [0, -1, 0], "breakdown_rho", 1),
    # the alpha denominator (r^, s_1) = 0 with rho_1 != 0
    "alpha_i0": ([[-1, -2, 1], [1, -1, 1], [1, -2, 1]], [1, 0, 0], "breakdown_alpha", 1),
}


def _mv(M, v):
    return [sum((M[i][j] * v[j] for j in range(len(v))), F(0)) for i in range(len(M))]


def _dot(a, b):
    return sum((x * y for x, y in zip(a, b)), F(0))


def alg2_exact(M, b, iters):
    """PAPER.md Algorithm 2 in exact rationals (readings R-1..R-3), x0 = 0.
    Per iteration i: omega, rho' = (r^, r_{i+1}), rr = (r_{i+1}, r_{i+1}),
    beta, d (the l.82 denominator), alpha', and x, r.  Stops after the first
    zero divisor (omega = 0, rho' = 0, d = 0) or r' = 0."""
    M = [[F(v) for v in row] for row in M]
    b = [F(v) for v in b]
    x = [F(0)] * len(b)
    r = list(b)
    rh = list(r)
    w = _mv(M, r)
    t = _mv(M, w)
    rho = _dot(rh, r)
    a = rho / _dot(rh, w)
    out = []
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
        rhon = _dot(rh, rn)
        e = dict(i=i, alpha=a, omega=om, rho1=rhon, rr=_dot(rn, rn), x=list(x), r=list(rn), rho0=_dot(rh, rh))
        out.append(e)
        if all(c == 0 for c in rn) or om == 0 or rhon == 0:
            break
        beta = (a / om) * rhon / rho
        d = _dot(rh, w) + beta * _dot(rh, s) - beta * om * _dot(rh, z)
        e.update(beta=beta, d=d)
        if d == 0:
            break
        a = rhon / d
        rho = rhon
        r = rn
    return out


def is_short_dyadic(f: F, bits: int = 50) -> bool:
    d = f.denominator
    return d & (d - 1) == 0 and abs(f.numerator) < (1 << bits)


def tile(M, b, m: int) -> tuple[gen.CSR, np.ndarray]:
    """m block-diagonal copies of the small system (zero entries not stored)."""
    M = np.asarray(M, np.float64)
    k = M.shape[0]
    rp, cols, vals = [0], [], []
    for blk in range(m):
        for i in range(k):
            nz = np.nonzero(M[i])[0]
            cols.extend((blk * k + nz).tolist())
            vals.extend(M[i, nz].tolist())
            rp.append(len(cols))
    A = gen.CSR(m * k, np.array(rp, np.int32), np.array(cols, np.int32), np.array(vals, np.float64),
                name=f"tile{k}x{m}", rhs="given")
    A.b = np.tile(np.asarray(b, np.float64), m)
    return A, A.b


def _ratio(num: F, rho0: F, rr: F) -> float:
    """|num| / (sqrt(rho0) sqrt(rr)), from the exact squares."""
    return math.sqrt(float(num * num / (rho0 * rr)))


def eps_for(M, b, kind: str, at: int, margin: float = 1e-6) -> float | None:
    """A breakdown_eps for which the R-11 threshold stops Algorithm 2 with
    breakdown_<kind> at iteration index `at` (iterations = at + 1) of the
    exact run, or None if no such eps exists for this system.  Earlier
    iterations need c_rho(i), c_d(i) > eps; at `at`: kind 'rho' needs
    c_rho(at) < eps, kind 'alpha' c_d(at) < eps < c_rho(at)."""
    tr = alg2_exact(M, b, at + 1)
    if len(tr) <= at or any("d" not in e for e in tr[:at + 1]):
        return None
    lo_bound = math.inf
    for e in tr[:at]:
        lo_bound = min(lo_bound, _ratio(e["rho1"], e["rho0"], e["rr"]), _ratio(e["d"], e["rho0"], e["rr"]))
    e = tr[at]
    crho = _ratio(e["rho1"], e["rho0"], e["rr"])
    cd = _ratio(e["d"], e["rho0"], e["rr"])
    if kind == "rho":
        lo, hi = crho, lo_bound
    else:
        lo, hi = cd, min(lo_bound, crho)
    if not lo * (1 + 20 * margin) < hi * (1 - 20 * margin):
        return None
    return lo * (1 + 10 * margin)


def _pmin(a, b):
    m = (a != 0) & (b != 0)
    return np.min(np.abs(a[m] * b[m])) if m.any() else np.inf


def product_minima(oracle, A, b, max_iter):
    """Smallest |fl(x_k y_k)| (x_k, y_k != 0) of each dot phase of the
    UNSCALED run, in execution order: ('I', -1, m) for the four init dots,
    then ('A', i, m) over (q,y),(y,y),(r^,s),(r^,z) and ('B', i, m) over
    (r^,r'),(r^,w'),(r',r') for i = 0, 1, ..."""
    O = oracle.PBiCGStab(A, b=b, tol=0.0, max_iter=max_iter)
    rh = O.vec("rh")
    out = [("I", -1, min(_pmin(b, b), _pmin(rh, O.vec("r")), _pmin(rh, O.vec("w")), _pmin(O.vec("r"), O.vec("r"))))]
    xs = [O.vec("x")]
    for i in range(max_iter):
        O.step()
        q, y, s, z = (O.vec(k) for k in "qysz")
        out.append(("A", i, min(_pmin(q, y), _pmin(y, y), _pmin(rh, s), _pmin(rh, z))))
        r, w = O.vec("r"), O.vec("w")
        out.append(("B", i, min(_pmin(rh, r), _pmin(rh, w), _pmin(r, r))))
        xs.append(O.vec("x"))
        if O.status != oracle.RUNNING:
            break
    return out, O.history(), xs


def range_case(oracle, A, b, phase: str, max_iter: int = 60, min_i: int = 1):
    """Choose k so that the run with b * 2^-k first meets a product below
    2^-960 (R-9) in `phase` ('A' or 'B') of an iteration i >= min_i.
    Returns (k, i, unscaled history, unscaled x after each iteration)."""
    seq, H, xs = product_minima(oracle, A, b, max_iter)
    for k in range(540, 399, -1):
        T = 2.0 ** (2 * k - 960)  # m * 2^-2k < 2^-960  <=>  m < T
        first = next(((ph, i) for ph, i, m in seq if m < T), None)
        if first is None:
            continue
        if first[0] == phase and first[1] >= min_i:
            return k, first[1], H, xs
    return None
