"""GPU parity for the rare paths of the streaming kernels' exact accumulator
(exblas.cuh ExAccT): products far below a thread's running sums (the warp
spill queue and the cold levels), superaccumulator deposits, magnitudes that
sweep across the exponent range, the top and bottom of the fast zone, and
many products per thread -- each compared bit for bit with the oracle's EXDOT
(correctly rounded for any input).

Sizes: the EXDOT grid is one CTA per SM x 12 consumer warps, so 2^26
elements give ~1,180 products per thread."""
import struct

import numpy as np
import pytest

import gen
import oracle

pytestmark = pytest.mark.gpu


def bits(v):
    return struct.unpack("<Q", struct.pack("<d", v))[0]


@pytest.fixture(scope="module")
def pb():
    import torch
    assert torch.cuda.is_available()
    import paper_2404_13216_b200 as pb
    return pb


def check(pb, x, y):
    import torch
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    want, wf = oracle.exdot(x, y)
    got, gf = pb.exdot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    assert bool(wf & oracle.F_RANGE) == bool(gf & pb.FLAG_RANGE), (wf, gf)
    assert bits(got) == bits(want), (x.size, got, want, wf)
    return got


def test_many_equal_products(pb):
    # every product positive and equal: the running sums grow through many
    # binades while the new products stay put
    n = 1 << 26
    x = np.full(n, 1.0 - 2.0 ** -52)
    y = np.full(n, 1.0 + 2.0 ** -30)
    assert check(pb, x, y) == oracle.exdot(x, y)[0]


def test_many_products_mixed(pb):
    n = (1 << 26) + 5
    x = gen.uniform(n, 11) * 2.0 ** 20
    y = gen.uniform(n, 12)
    check(pb, x, y)


@pytest.mark.parametrize("order", ["ascending", "descending", "sawtooth"])
def test_magnitude_sweeps(pb, order):
    # magnitudes sweep 900 binades along the index: the running sums are
    # overtaken tile after tile (ascending), or every new product falls far
    # below them (descending), or both (sawtooth)
    n = 1 << 20
    e = np.linspace(-450, 450, n)
    if order == "descending":
        e = e[::-1]
    elif order == "sawtooth":
        e = np.tile(np.linspace(-450, 450, 4096), n // 4096)
    x = np.ldexp(gen.uniform(n, 3), np.floor(e).astype(int))
    y = np.ldexp(1.0 + gen.uniform(n, 4, 0.0, 1.0), np.floor(e).astype(int))
    check(pb, x, y)


@pytest.mark.parametrize("seed", range(4))
def test_far_below_running_sums(pb, seed):
    # one large product per 64 elements, the rest 60-240 binades below it:
    # spills every batch, cold levels, superaccumulator deposits
    n = 1 << 21
    x = gen.loguniform(n, seed, -200, -60)
    x[::64] = gen.uniform(n // 64, seed + 10) * 2.0 ** 40
    y = gen.uniform(n, seed + 20)
    check(pb, x, y)


def test_top_of_fast_zone(pb):
    # products just below the R-9 fast-zone limit 2^1000, with cancellation
    n = 8192
    x = np.full(n, 2.0 ** 499) * np.where(np.arange(n) % 2 == 0, 1.0, -1.0)
    y = np.full(n, 1.75 * 2.0 ** 499)
    y[::7] *= 0.5
    x[-1] = 3.0
    check(pb, x, y)


def test_bottom_of_fast_zone(pb):
    # products just above 2^-960 (the lowest products whose e is exact)
    n = 1 << 18
    x = np.ldexp(1.0 + gen.uniform(n, 5, 0.0, 1.0), -480)
    y = np.ldexp(gen.uniform(n, 6), -470)
    check(pb, x, y)


def test_ill_conditioned_many_per_thread(pb):
    # GenDot blocks (condition ~1e30) at ~1,180 products per thread
    x, y = gen.ill_pair(1 << 26, seed=17, block=1 << 16)
    check(pb, x, y)
