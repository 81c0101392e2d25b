"""GPU parity: the CUDA ExBLAS dot (through the C ABI `exdot`) against the
oracle's EXDOT, bit for bit (BASELINE.json north_star: "The GPU ExBLAS dots
must match it bit-exactly")."""
import math
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


def gpu_exdot(pb, x, y, handle=None):
    import torch
    xt = torch.from_numpy(np.ascontiguousarray(x, np.float64)).cuda()
    yt = torch.from_numpy(np.ascontiguousarray(y, np.float64)).cuda()
    return pb.exdot(xt, yt, handle=handle)


def check(pb, x, y, handle=None):
    want, wf = oracle.exdot(x, y)
    got, gf = gpu_exdot(pb, x, y, handle)
    # flag contract (include/pbicgstab.h): NONFINITE iff an input is NaN/Inf;
    # otherwise RANGE iff a nonzero product leaves the fast pass's exact zone (R-9)
    assert bool(wf & oracle.F_NONFINITE) == bool(gf & pb.FLAG_NONFINITE), (wf, gf)
    if not wf & oracle.F_NONFINITE:
        assert bool(wf & oracle.F_RANGE) == bool(gf & pb.FLAG_RANGE), (wf, gf)
        # single GPU: RANGE dots go through the full-range pass (NEXT-4) and
        # are exact too; the oracle's value is exact over the whole range
        if wf == 0 or handle is None:
            assert bits(got) == bits(want), (len(x), got, want, wf)
    return got


def test_spec_examples(pb):
    assert gpu_exdot(pb, [1e16, 1.0, -1e16], [1, 1, 1]) == (1.0, 0)
    v, f = gpu_exdot(pb, [], [])
    assert bits(v) == bits(0.0) and f == 0
    v, _ = gpu_exdot(pb, [-0.0, 3.0, -3.0], [1.0, 1.0, 1.0])
    assert bits(v) == bits(0.0)
    assert gpu_exdot(pb, np.full(10 ** 6, 0.1), np.ones(10 ** 6))[0] == 100000.0
    assert gpu_exdot(pb, [1.0, 2.0 ** -53], [1, 1])[0] == 1.0
    assert gpu_exdot(pb, [1.0 + 2.0 ** -52, 2.0 ** -53], [1, 1])[0] == 1.0 + 2.0 ** -51
    for i in range(5):
        for j in range(5):
            assert gpu_exdot(pb, np.eye(5)[i], np.eye(5)[j])[0] == (1.0 if i == j else 0.0)


def test_edge_values(pb):
    u = 2.0 ** -52
    check(pb, [(1 + u) * 2.0 ** -480, -(1 + 2 * u) * 2.0 ** -480], [(1 + u) * 2.0 ** -480, 2.0 ** -480])
    # the same magnitudes with negative sums: the rounding works on the
    # two's complement superaccumulator (negation, ties, subnormals)
    check(pb, [-(1 + u) * 2.0 ** -480, (1 + 2 * u) * 2.0 ** -480], [(1 + u) * 2.0 ** -480, 2.0 ** -480])
    for sgn in (1.0, -1.0):
        check(pb, [sgn, sgn * 2.0 ** -53], [1.0, 1.0])                      # tie to even
        check(pb, [sgn * (1.0 + 2.0 ** -52), sgn * 2.0 ** -53], [1.0, 1.0])  # tie to even, rounds away
        check(pb, [sgn, sgn * 2.0 ** -53, sgn * 2.0 ** -300], [1.0, 1.0, 1.0])  # sticky far below
        check(pb, [sgn * 2.0 ** 900, -sgn * 2.0 ** 900, sgn * 3.0], [2.0 ** 90, 2.0 ** 90, 2.0 ** -900])
        check(pb, [sgn * 2.0 ** 400] * 8, [2.0 ** 599] * 8)                 # near overflow, in range
        check(pb, [sgn * (2.0 - 2.0 ** -52) * 2.0 ** 499] * 2, [2.0 ** 499, 2.0 ** 499])
    # range zone and non-finite flags mirror the oracle (R-9)
    check(pb, [2.0 ** -1074], [1.0])
    check(pb, [2.0 ** -480], [2.0 ** -481])
    check(pb, [2.0 ** 500], [2.0 ** 500])
    check(pb, [0.0, 2.0 ** -1074], [2.0 ** -1074, 0.0])
    check(pb, [1.0, math.nan], [1.0, 1.0])
    check(pb, [math.inf, 1.0], [0.0, 1.0])


@pytest.mark.parametrize("n", [1, 2, 3, 31, 32, 33, 255, 256, 257, 511, 1000, 4097, 65537, 1 << 18, (1 << 20) + 3])
def test_sizes_ragged(pb, n):
    # spans several tiles, odd lengths exercise the scalar tail and the
    # unaligned path
    x = gen.uniform(n, 1)
    y = gen.uniform(n, 2)
    check(pb, x, y)
    check(pb, x[1:], y[1:])  # 8-byte misaligned start


@pytest.mark.parametrize("seed", range(12))
def test_random_distributions(pb, seed):
    n = 5000 + 777 * seed
    kind = seed % 4
    if kind == 0:
        x, y = gen.loguniform(n, seed, -100, 100), gen.loguniform(n, seed + 99, -100, 100)
    elif kind == 1:
        x, y = gen.ill_pair(n - n % 2, seed=seed, block=1024)
    elif kind == 2:  # heavy cancellation
        x = gen.uniform(n, seed) * 2.0 ** 40
        x = np.concatenate([x, -x, gen.uniform(7, seed)])
        y = np.concatenate([gen.uniform(n, seed + 1), gen.uniform(n, seed + 1), gen.uniform(7, seed + 3)])
    else:  # sparse-ish vectors with exact zeros (like r0 of the stencil configs)
        x = gen.uniform(n, seed)
        x[::3] = 0.0
        y = gen.uniform(n, seed + 5)
    check(pb, x, y)


def test_permutation_invariance(pb):
    x, y = gen.ill_pair(1 << 16, seed=21, block=1 << 14)
    ref = bits(gpu_exdot(pb, x, y)[0])
    rng = np.random.default_rng(0)
    for _ in range(5):
        p = rng.permutation(x.size)
        assert bits(gpu_exdot(pb, x[p], y[p])[0]) == ref


@pytest.mark.parametrize("kind", ["well", "ill"])
def test_full_size_2_26(pb, kind):
    # BASELINE.json configs[1] at n = 2^26, in the launch configuration bench.py times
    n = 1 << 26
    if kind == "well":
        x, y = gen.uniform(n, 1), gen.uniform(n, 2)
    else:
        x, y = gen.ill_pair(n, seed=3)
    check(pb, x, y)


def test_virtual_rank_partition_invariance(pb):
    # the cross-rank path (per-rank superaccumulators, int64 sum, one rounding)
    # on one GPU: identical bits for 1..8 virtual ranks
    import torch
    x, y = gen.ill_pair(1 << 17, seed=5, block=1 << 12)
    want = oracle.exdot(x, y)[0]
    A = gen.stencil(2, 16, 10.0)
    for V in (2, 3, 4, 8):
        S = pb.Solver(A.row_ptr, A.col, A.val, A.n, virtual_ranks=V)
        got, f = gpu_exdot(pb, x, y, handle=S)
        assert f == 0 and bits(got) == bits(want), V
        S.close()


def test_on_device_result_and_plain_dot(pb):
    import torch
    n = 1 << 20
    x = torch.from_numpy(gen.uniform(n, 7)).cuda()
    y = torch.from_numpy(gen.uniform(n, 8)).cuda()
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    fl = torch.zeros(1, dtype=torch.int32, device="cuda")
    pb.exdot(x, y, on_device=True, out=out, flags_out=fl)
    torch.cuda.synchronize()
    want = oracle.exdot(x.cpu().numpy(), y.cpu().numpy())[0]
    assert bits(out.item()) == bits(want) and fl.item() == 0
    p = pb.dot_plain(x, y)
    torch.cuda.synchronize()
    assert abs(p.item() - want) <= 1e-12 * float(torch.sum(torch.abs(x * y)))


def test_nccl_single_rank_handle(pb):
    # distributed EXDOT path (per-rank superaccumulator, ncclAllReduce int64,
    # finalize) with a 1-rank communicator
    x, y = gen.ill_pair(1 << 16, seed=9, block=1 << 12)
    A = gen.stencil(2, 16, 10.0)
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n, force_nccl=True)
    got, f = gpu_exdot(pb, x, y, handle=S)
    assert f == 0 and bits(got) == bits(oracle.exdot(x, y)[0])
    S.close()


@pytest.mark.parametrize("kind,n", [("well", 1 << 22), ("ill", 1 << 20), ("ragged", 100_003), ("unaligned", 4_097)])
def test_comm_only_handle(pb, kind, n):
    # comm-only handle (pbicgstab_setup with A = NULL) through
    # the NCCL dataflow (1-rank communicator): the rank's slice goes through
    # the TMA stream kernel (finalize = 0), the words through ncclAllReduce
    # int64, then one rounding -- bit-exact; and without NCCL (local handle)
    import torch
    if kind == "ill":
        x, y = gen.ill_pair(n, seed=9, block=1 << 12)
    else:
        x, y = gen.uniform(n, 3), gen.uniform(n, 4)
    want = oracle.exdot(x, y)[0]
    for force in (True, False):
        C = pb.Comm(force_nccl=force)
        xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
        if kind == "unaligned":  # 8-byte aligned slices: the generic kernel
            xt, yt = torch.from_numpy(np.concatenate([[0.0], x])).cuda()[1:], torch.from_numpy(np.concatenate([[0.0], y])).cuda()[1:]
        got, f = C.exdot(xt, yt)
        assert f == 0 and bits(got) == bits(want), (kind, force)
        C.close()


# ---- full-range EXDOT: products outside the fast zone ----

def test_full_range_underflow_zone(pb):
    # products below 2^-960: TwoProd is inexact there, the full-range pass is not
    t = 2.0 ** -540
    check(pb, [t, t], [t, -t * (1 + 2.0 ** -52)])              # cancels to a tiny exact difference
    check(pb, [2.0 ** -1074, 2.0 ** -1074], [0.5, 0.5])        # survey example: exact 2^-1074
    check(pb, [2.0 ** -1074] * 3, [0.5, 0.5, 0.5])             # 1.5 * 2^-1074: tie -> even
    check(pb, [2.0 ** -600] * 64, [2.0 ** -480] * 64)          # sum lands in the subnormals
    check(pb, [1.0, 2.0 ** -600], [1.0, 2.0 ** -600])          # far below: rounds away (sticky)
    check(pb, [2.0 ** -1022, -2.0 ** -1022], [2.0 ** -52, 2.0 ** -53])


def test_full_range_overflow_zone(pb):
    big = 2.0 ** 520
    check(pb, [big, -big, 3.0], [big, big, 1.0])               # huge products cancel exactly
    check(pb, [2.0 ** 1000, 2.0 ** 1000], [2.0 ** 23, -2.0 ** 23 + 1])
    v, f = gpu_exdot(pb, [2.0 ** 1000] * 4, [2.0 ** 23] * 4)  # exact sum 2^1025: overflows to +inf
    assert v == math.inf and f & pb.FLAG_RANGE
    assert oracle.exdot([2.0 ** 1000] * 4, [2.0 ** 23] * 4)[0] == math.inf


@pytest.mark.parametrize("seed", range(6))
def test_full_range_random(pb, seed):
    # exponents over the whole binary64 range: products from 2^-2140 to 2^1000
    rng = np.random.default_rng(seed)
    n = 3000 + 1000 * seed
    ex = rng.integers(-1070, 500, n)
    ey = rng.integers(-1070, 500, n)
    x = np.ldexp(rng.uniform(1, 2, n) * rng.choice([-1.0, 1.0], n), ex)
    y = np.ldexp(rng.uniform(1, 2, n) * rng.choice([-1.0, 1.0], n), ey)
    if seed % 2:  # keep only the small ones: the result is decided far below 2^-960
        keep = (ex + ey) < -1000
        x, y = x[keep], y[keep]
    check(pb, x, y)


@pytest.mark.parametrize("where", ["one", "spread", "all"])
def test_full_range_many_ctas(pb, where):
    # full-range pass across CTAs: the flagged CTAs recompute their own
    # elements into the extended accumulator, the others keep their fast
    # words; the last CTA adds both and rounds once
    n = (1 << 21) + 37
    x, y = gen.uniform(n, 11), gen.uniform(n, 12)
    rng = np.random.default_rng(7)
    if where == "all":
        x, y = gen.loguniform(n, 5, -540, 0), gen.loguniform(n, 6, -540, 0)
    else:
        idx = [n // 3] if where == "one" else rng.choice(n, 40, replace=False)
        for k, i in enumerate(idx):
            x[i] = 2.0 ** -700 * (1 + k / 64)
            y[i] = -(2.0 ** -300) if k % 2 else 2.0 ** -301
        # the exact sum is tiny: cancel the fast part down to O(1e-300)
        x[0] = 0.0
    check(pb, x, y)
    # the same through the general (unaligned) kernel: its CTAs walk strided pairs
    import torch
    xt = torch.from_numpy(np.concatenate([[0.0], x])).cuda()[1:]
    yt = torch.from_numpy(np.concatenate([[0.0], y])).cuda()[1:]
    want, wf = oracle.exdot(x, y)
    got, gf = pb.exdot(xt, yt)
    assert bits(got) == bits(want) and bool(gf & pb.FLAG_RANGE) == bool(wf & oracle.F_RANGE), (got, want, gf, wf)
    # cancellation: the fast words and the extended sums meet in the low bits
    x2 = np.concatenate([x, -x, [2.0 ** -600]])
    y2 = np.concatenate([y, y, [-(2.0 ** -450)]])
    assert check(pb, x2, y2) == -(2.0 ** -1050)


def test_full_range_nonfinite_in_one_cta(pb):
    n = 1 << 21
    x, y = gen.uniform(n, 13), gen.uniform(n, 14)
    x[n // 2] = 2.0 ** -700
    y[n // 2] = 2.0 ** -400
    x[n - 5] = np.inf
    v, f = gpu_exdot(pb, x, y)
    assert f & pb.FLAG_NONFINITE
    check(pb, x, y)


@pytest.mark.parametrize("where", ["spread", "all", "overflow_zone", "random"])
def test_full_range_distributed(pb, where):
    # full range per rank (R-24): each rank's flagged CTAs correct their
    # products into extended words, which are summed across ranks (int64)
    # with the fast words and rounded once -- virtual ranks, the comm-only
    # handle through NCCL (1-rank communicator), bit-exact against the oracle
    import torch
    n = (1 << 20) + 11
    rng = np.random.default_rng(3)
    if where == "all":
        x, y = gen.loguniform(n, 5, -540, 0), gen.loguniform(n, 6, -540, 0)
    elif where == "random":
        n = 20_000
        ex, ey = rng.integers(-1070, 500, n), rng.integers(-1070, 500, n)
        x = np.ldexp(rng.uniform(1, 2, n) * rng.choice([-1.0, 1.0], n), ex)
        y = np.ldexp(rng.uniform(1, 2, n) * rng.choice([-1.0, 1.0], n), ey)
    else:
        x, y = gen.uniform(n, 11), gen.uniform(n, 12)
        idx = rng.choice(n, 40, replace=False)
        for k, i in enumerate(idx):
            if where == "spread":
                x[i], y[i] = 2.0 ** -700 * (1 + k / 64), (-(2.0 ** -300) if k % 2 else 2.0 ** -301)
            else:  # products above 2^1000 that cancel: the FPE-overflow (poisoned) path
                x[i], y[i] = 2.0 ** 510 * (1 + k / 64), (2.0 ** 500 if k % 2 == 0 else -(2.0 ** 500))
                if k % 2:
                    x[i] = x[idx[k - 1]]
    want, wf = oracle.exdot(x, y)
    assert np.isfinite(want)
    xt, yt = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    A = gen.stencil(2, 16, 10.0)
    for V in (2, 3):
        S = pb.Solver(A.row_ptr, A.col, A.val, A.n, virtual_ranks=V)
        got, f = pb.exdot(xt, yt, handle=S)
        assert bits(got) == bits(want), (where, V, got, want)
        S.close()
    C = pb.Comm(force_nccl=True)
    got, f = C.exdot(xt, yt)
    assert bits(got) == bits(want), (where, "comm", got, want)
    C.close()
