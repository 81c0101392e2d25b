"""Pins for the oracle's SpMV (fixed left-to-right per-row FMA chain, SPEC.md
l.161-169, reading R-6) and for the input generators' structure."""
import struct
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle


def bits(v):
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def fr_fma(a, b, c):
    # one rounding of the exact a*b+c (CPython int/int division is correctly rounded)
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def test_identity_and_diag():
    # SPEC.md l.167-168
    I = gen.from_dense(np.eye(5))
    x = np.array([1.5, -2.0, 3.25, 0.1, 7.0])
    assert np.array_equal(oracle.spmv(I, x), x)
    D = gen.from_dense(np.array([[2.0]]))
    assert oracle.spmv(D, [1.0])[0] == 2.0


def test_empty_row_is_plus_zero():
    A = gen.CSR(3, np.array([0, 1, 1, 2], np.int32), np.array([0, 2], np.int32), np.array([1.0, -1.0]))
    y = oracle.spmv(A, np.array([-0.0, 5.0, 0.0]))
    assert bits(y[1]) == bits(0.0)
    # y starts at +0.0: a single -0*... term gives fma(1,-0,+0) = +0
    assert bits(y[0]) == bits(0.0)


@pytest.mark.parametrize("seed", range(6))
def test_random_50x50_vs_fraction_fma_chain(seed):
    # random 50x50, 10% density, 0 ulp against a dense oracle in
    # the same order.  The chain here is evaluated with exact rationals and one
    # rounding per step, which pins both the order and the single-rounding FMA.
    rng = np.random.default_rng(seed)
    M = rng.uniform(-1, 1, (50, 50)) * (rng.uniform(0, 1, (50, 50)) < 0.1)
    M *= 2.0 ** rng.integers(-30, 30, (50, 50))
    A = gen.from_dense(M)
    x = rng.uniform(-1, 1, 50) * 2.0 ** rng.integers(-30, 30, 50)
    y = oracle.spmv(A, x)
    for i in range(50):
        acc = 0.0
        for j in range(50):
            if M[i, j] != 0.0:
                acc = fr_fma(M[i, j], x[j], acc)
        assert bits(y[i]) == bits(acc), i


def test_fma_not_two_roundings():
    # a case where fma differs from mul-then-add: (1+2^-30)^2 - (1+2^-29)
    a = 1.0 + 2.0 ** -30
    A = gen.CSR(1, np.array([0, 2], np.int32), np.array([0, 1], np.int32), np.array([-(1.0 + 2.0 ** -29), a]))
    y = oracle.spmv(A, np.array([1.0, a]))[0]
    assert y == 2.0 ** -60  # exact; mul-then-add would give 0.0


def test_row_partition_invariance():
    # spmv is bitwise identical under any row partition
    A = gen.stencil(3, 12, 100.0)
    x = gen.uniform(A.n, 9)
    y = oracle.spmv(A, x)
    for P in (2, 3, 8):
        parts = []
        for p in range(P):
            r0, r1 = A.n * p // P, A.n * (p + 1) // P
            parts.append(oracle.spmv(A.rows(r0, r1), x))
        assert np.array_equal(np.concatenate(parts).view(np.uint64), y.view(np.uint64))


def test_stencil_structure_and_rowsums():
    for d, N, Pe in [(2, 64, 10.0), (3, 16, 100.0)]:
        A = gen.stencil(d, N, Pe)
        assert A.nnz == (2 * d + 1) * N ** d - 2 * d * N ** (d - 1)
        assert np.all(np.diff(A.row_ptr) >= d + 1)
        for i in range(A.n):
            c = A.col[A.row_ptr[i]:A.row_ptr[i + 1]]
            assert np.all(np.diff(c) > 0)
        b = oracle.spmv(A, np.ones(A.n))
        # row sums by exact rationals: interior rows of the upwind stencil sum to 0
        h = 1.0 / (N + 1)
        hc = h * Pe
        lo, up, dg = -(1.0 + hc), -1.0, float(2 * d) + d * hc
        assert set(np.unique(A.val)) == {lo, up, dg}
        interior = [i for i in range(A.n) if A.row_ptr[i + 1] - A.row_ptr[i] == 2 * d + 1]
        if d == 2:
            assert np.all(b[interior] == 0.0)  # checked in SURVEY.md App. A
    assert gen.stencil(2, 64, 10.0).nnz == 20224
    assert gen.stencil(3, 128, 100.0).nnz == 14581760


def test_random_banded_structure():
    n = 1 << 15
    A = gen.random_banded(n, seed=42)
    lens = np.diff(A.row_ptr)
    assert lens.min() >= 5 and lens.max() <= 200
    assert abs(lens.mean() - 27.0) < 0.2
    rows = np.repeat(np.arange(n), lens)
    assert np.all(np.abs(A.col - rows) <= 5000)
    for i in range(0, n, 997):
        s, e = A.row_ptr[i], A.row_ptr[i + 1]
        c, v = A.col[s:e], A.val[s:e]
        assert np.all(np.diff(c) > 0) and i in c
        off = v[c != i]
        asum = 0.0
        for t in off:
            asum = asum + abs(t)
        assert v[c == i][0] == 1.2 * asum
    B = gen.random_banded(n, seed=42)
    assert np.array_equal(A.col, B.col) and np.array_equal(A.val, B.val)
