"""Pins for the oracle's EXDOT (oracle/oracle.c orc_exdot / orc_acc_*).

EXDOT(x,y) is defined as the binary64 nearest (ties-to-even) to the exact
real sum x_k*y_k (§2 l.95).  Nothing here
re-implements the oracle's big-integer accumulator: values are pinned against
``fractions.Fraction`` brute force (CPython's int/int true division is
correctly rounded, ties-to-even, subnormals included), ``math.fsum`` (an
independent correctly-rounded sum of doubles), the worked examples SPEC.md
gives, and invariants (permutation, partition, merge order).
"""
import math
import struct
from fractions import Fraction

import numpy as np
import pytest

import gen
import oracle


def bits(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def exact(x, y) -> Fraction:
    return sum((Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y)), Fraction(0))


def rn(f: Fraction) -> float:
    return float(f)  # correctly rounded, ties-to-even


def check(x, y):
    got, flags = oracle.exdot(x, y)
    want = rn(exact(x, y))
    assert bits(got) == bits(want), (got, want)
    return got, flags


# --- SPEC.md worked examples --------------------------------------------------

def test_spec_cancellation_example():
    # x=[1e16,1,-1e16], y=[1,1,1] -> Reproducible 1.0 (Sequential 0.0)
    v, f = oracle.exdot([1e16, 1.0, -1e16], [1.0, 1.0, 1.0])
    assert v == 1.0 and f == 0
    assert oracle.dot_seq([1e16, 1.0, -1e16], [1.0, 1.0, 1.0]) == 0.0


def test_spec_empty_is_plus_zero():
    # SPEC.md l.69 / l.105: empty sum -> 0.0 ; reading R-8: exact zero -> +0.0
    v, f = oracle.exdot([], [])
    assert bits(v) == bits(0.0) and f == 0
    v, _ = oracle.exdot([-0.0, 3.0, -3.0], [1.0, 1.0, 1.0])
    assert bits(v) == bits(0.0)


def test_spec_million_tenths():
    # 10^6 copies of 0.1 -> RN(10^6 * fl(0.1)) = 100000.0
    n = 10 ** 6
    v, _ = oracle.exdot(np.full(n, 0.1), np.ones(n))
    assert v == rn(n * Fraction(0.1)) == 100000.0


def test_spec_ties_to_even():
    # 1 + 2^-53 -> 1.0 ; (1+2^-52) + 2^-53 -> 1 + 2^-51
    assert oracle.exdot([1.0, 2.0 ** -53], [1.0, 1.0])[0] == 1.0
    assert oracle.exdot([1.0 + 2.0 ** -52, 2.0 ** -53], [1.0, 1.0])[0] == 1.0 + 2.0 ** -51
    # a tie that rounds down to even and one below/above the tie
    assert oracle.exdot([1.0, 2.0 ** -53, 2.0 ** -100], [1, 1, 1])[0] == 1.0 + 2.0 ** -52
    assert oracle.exdot([1.0, 2.0 ** -53, -(2.0 ** -100)], [1, 1, 1])[0] == 1.0


def test_spec_unit_vectors():
    # dot(e_i, e_j) = delta_ij
    n = 7
    for i in range(n):
        for j in range(n):
            ei, ej = np.eye(n)[i], np.eye(n)[j]
            assert oracle.exdot(ei, ej)[0] == (1.0 if i == j else 0.0)


def test_smallest_subnormal_preserved_but_flagged():
    # an accumulator holding exactly 2^-1074 rounds to 2^-1074.
    a = oracle.Acc().add(2.0 ** -1074)
    assert a.round() == 2.0 ** -1074 and a.flags == 0
    # As a product this is in the GPU TwoProd underflow zone (reading R-9):
    v, f = oracle.exdot([2.0 ** -1074], [1.0])
    assert v == 2.0 ** -1074 and f & oracle.F_RANGE
    # survey example: [2^-1074,2^-1074].[1/2,1/2] is exactly 2^-1074
    v, f = oracle.exdot([2.0 ** -1074] * 2, [0.5, 0.5])
    assert v == 2.0 ** -1074 and f & oracle.F_RANGE


def test_subnormal_result_from_cancellation_is_exact():
    u = 2.0 ** -52
    x = [(1 + u) * 2.0 ** -480, -(1 + 2 * u) * 2.0 ** -480]
    y = [(1 + u) * 2.0 ** -480, 2.0 ** -480]
    v, f = check(x, y)
    assert v == 2.0 ** -1064 and f == 0  # products are >= 2^-960: no range flag


def test_overflow_gives_inf_and_range():
    v, f = oracle.exdot([1e308] * 4, [10.0] * 4)
    assert v == math.inf and f & oracle.F_RANGE
    v, f = oracle.exdot([-1e308] * 4, [10.0] * 4)
    assert v == -math.inf and f & oracle.F_RANGE


def test_range_rule_thresholds():
    # reading R-9: flag iff x,y != 0 and |fl(x*y)| < 2^-960 or >= 2^1000
    assert oracle.exdot([2.0 ** -480], [2.0 ** -480])[1] == 0
    assert oracle.exdot([2.0 ** -480], [2.0 ** -481])[1] & oracle.F_RANGE
    assert oracle.exdot([2.0 ** 500], [2.0 ** 499])[1] == 0
    assert oracle.exdot([2.0 ** 500], [2.0 ** 500])[1] & oracle.F_RANGE
    assert oracle.exdot([0.0, 2.0 ** -1074], [2.0 ** -1074, 0.0])[1] == 0  # zero products are fine


def test_nonfinite_flag():
    assert oracle.exdot([1.0, math.nan], [1.0, 1.0])[1] & oracle.F_NONFINITE
    assert oracle.exdot([1.0, 2.0], [math.inf, 1.0])[1] & oracle.F_NONFINITE


# --- brute force against Fraction ------------------------------------------------

@pytest.mark.parametrize("seed", range(40))
def test_random_vs_fraction(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 300))
    kind = seed % 4
    if kind == 0:
        x, y = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    elif kind == 1:  # log-uniform magnitudes spanning 1e+-30
        x = gen.loguniform(n, seed, -100, 100)
        y = gen.loguniform(n, seed + 1000, -100, 100)
    elif kind == 2:  # heavy cancellation
        x = rng.uniform(-1, 1, n) * 2.0 ** rng.integers(-60, 60, n)
        y = rng.uniform(-1, 1, n)
        x = np.concatenate([x, x])
        y = np.concatenate([y, -y * (1 + 2.0 ** -40)])
    else:  # GenDot-style ill-conditioned pairs
        m = max(8, n - n % 2)
        x, y = gen.ill_pair(m, seed=seed, block=m)
    check(x, y)


def test_fsum_special_case():
    # EXDOT(x, ones) is the correctly rounded sum of x, which math.fsum computes
    # independently (Shewchuk's algorithm).
    for seed in range(10):
        x = gen.loguniform(5000, seed, -40, 40)
        assert bits(oracle.exdot(x, np.ones_like(x))[0]) == bits(math.fsum(x))


def test_ten_thousand_loguniform_vs_fraction():
    # random 10^4-element accumulation equals the big-integer oracle
    x = gen.loguniform(10_000, 7, -100, 100)
    y = gen.loguniform(10_000, 8, -100, 100)
    check(x, y)


def test_ill_conditioned_generator_condition():
    # The C2-ILL generator reaches cond ~ 1e30 (BASELINE.json configs[1]);
    # cond = 2 sum|x y| / |sum x y| with both sums exact.
    x, y = gen.ill_pair(1 << 12, seed=3, block=1 << 12)
    ex = exact(x, y)
    ab = sum(abs(Fraction(a) * Fraction(b)) for a, b in zip(x, y))
    cond = float(2 * ab / abs(ex))
    assert cond > 1e25
    assert oracle.exdot(x, y)[0] == rn(ex)
    lx = np.log2(np.abs(x[x != 0]))
    assert lx.min() < -150 and lx.max() > 150  # exponents spread over ~[-200,200]


# --- invariants --------------------------------------------------------------------

def test_permutation_invariance():
    rng = np.random.default_rng(1)
    x = gen.loguniform(20_000, 11, -60, 60)
    y = gen.loguniform(20_000, 12, -60, 60)
    ref = bits(oracle.exdot(x, y)[0])
    for _ in range(20):
        p = rng.permutation(x.size)
        assert bits(oracle.exdot(x[p], y[p])[0]) == ref


@pytest.mark.parametrize("nparts", [1, 2, 4, 8, 16, 64])
def test_partition_and_merge_order_invariance(nparts):
    # SPEC.md l.110 (partition invariance), l.79 (tree shapes)
    rng = np.random.default_rng(nparts)
    x, y = gen.ill_pair(1 << 14, seed=5, block=1 << 12)
    ref = bits(oracle.exdot(x, y)[0])
    for _ in range(5):
        order = rng.permutation(nparts)
        assert bits(oracle.exdot_parts(x, y, nparts, order)[0]) == ref


def test_merge_identity_and_commutativity():
    # SPEC.md l.77-78
    a = oracle.Acc().add(5.0)
    assert a.merge(oracle.Acc()).round() == 5.0
    xs = gen.loguniform(200, 3, -30, 30)
    ys = gen.loguniform(200, 4, -30, 30)
    p, q = oracle.Acc(), oracle.Acc()
    for v in xs:
        p.add(v)
    for v in ys:
        q.add(v)
    p2, q2 = oracle.Acc(), oracle.Acc()
    for v in xs:
        p2.add(v)
    for v in ys:
        q2.add(v)
    assert bits(p.merge(q).round()) == bits(q2.merge(p2).round())
