"""Parity at the full BASELINE.json sizes, in the launch configuration
bench.py times (CUDA-graph chunks of iterate(), persistent TMA kernels).

The oracle is affordable for the first few iterations of C4/C5; beyond that
the checks are properties that hold at any size: identical bits for 1 rank,
4 virtual ranks and the NCCL dataflow (iteration counts of the
ExBLAS variant do not depend on the number of processes)."""
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


def gpu_run(pb, A, iters, **kw):
    import torch
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=iters + 8, **kw)
    b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
    S.start(b, tol=0.0, max_iter=iters + 4)
    S.iterate(iters)
    x = torch.zeros(A.n, dtype=torch.float64, device="cuda")
    r = S.finish(x)
    vecs = {k: S.vec(k) for k in ("r", "w", "t", "v", "s", "z")}
    H = S.history()
    S.close()
    return b.cpu().numpy(), x.cpu().numpy(), r, H, vecs


@pytest.mark.parametrize("name,iters", [("c5_3d256", 3), ("c4_rand4m", 2)])
def test_full_size_vs_oracle(pb, name, iters):
    A = gen.make_config(name)
    b, x, r, H, vecs = gpu_run(pb, A, iters)
    O = oracle.PBiCGStab(A, b=A.b if A.rhs == "given" else None, tol=0.0, max_iter=iters + 4)
    assert O.rc == 0
    assert np.array_equal(u64(b), u64(O.vec("b")))
    O.run(iters)
    assert r.iterations == O.iterations == iters
    assert np.array_equal(u64(H), u64(O.history()))
    assert np.array_equal(u64(x), u64(O.vec("x")))
    for k, v in vecs.items():  # every auxiliary vector of Alg. 2, bit for bit
        assert np.array_equal(u64(v), u64(O.vec(k))), k


def test_c5_partition_invariance(pb):
    A = gen.make_config("c5_3d256")
    ref = gpu_run(pb, A, 24)
    for kw in (dict(virtual_ranks=4), dict(force_nccl=True)):
        b, x, r, H, vecs = gpu_run(pb, A, 24, **kw)
        assert np.array_equal(u64(H), u64(ref[3])), kw
        assert np.array_equal(u64(x), u64(ref[1])), kw


def test_exdot_2_28_well(pb):
    import torch
    n = 1 << 28
    x, y = gen.uniform(n, 1), gen.uniform(n, 2)
    want, wf = oracle.exdot(x, y)
    got, gf = pb.exdot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    assert wf == 0 and gf == 0 and u64(got)[()] == u64(want)[()]


def test_exdot_2_28_ill(pb):
    # BASELINE.json configs[1] at its larger size, ill-conditioned (cond ~1e30)
    import torch
    n = 1 << 28
    x, y = gen.ill_pair(n, seed=3)
    want, wf = oracle.exdot(x, y)
    got, gf = pb.exdot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
    assert wf == 0 and gf == 0 and u64(got)[()] == u64(want)[()]


def test_c4_north_star_vs_plain_alg1(pb):
    # north_star: the final ||b - Ax||/||b|| agrees with a plain-double
    # BiCGStab (Alg. 1, the oracle's sequential dots) within 1e-10 --
    # on the full C4 config, solved to convergence on the GPU
    import torch
    A = gen.make_config("c4_rand4m")
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=256)
    x, r = S.solve(torch.from_numpy(A.b).cuda(), tol=1e-10, max_iter=250)
    S.close()
    assert r.status == pb.CONVERGED, r
    st, it, xb, _ = oracle.bicgstab(A, A.b, tol=1e-10, max_iter=250)
    assert st == oracle.CONVERGED
    tb = oracle.true_relres(A, A.b, xb)[0]
    tg = oracle.true_relres(A, A.b, x.cpu().numpy())[0]
    assert tg == r.relres_true  # the GPU's own true residual, bit for bit
    assert abs(r.relres_true - tb) <= 1e-10, (r.relres_true, tb, r.iterations, it)
