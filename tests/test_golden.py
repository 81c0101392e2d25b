"""Worked examples printed in /root/reference/SPEC.md, kept as text fixtures
under tests/golden/ (each line cites its SPEC.md line).  The oracle is checked
against them here (-m "not gpu"); the GPU path through the C ABI in the
gpu-marked tests at the bottom.  The paper's own printed numbers (Table 1
iteration counts) need the SuiteSparse matrices, which are not in this
container."""
import os
import struct

import numpy as np
import pytest

import gen
import oracle

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def num(s: str) -> float:
    s = s.strip()
    if "**" in s:  # powers of two, e.g. 2**-1074
        base, e = s.split("**")
        return float(base) ** int(e)
    return float(s)


def vec(s: str) -> np.ndarray:
    return np.array([num(v) for v in s.split(",") if v.strip()], np.float64)


def rows(name: str):
    out = []
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if line and not line.startswith("#"):
            out.append([f.strip() for f in line.split("|")])
    assert out, name
    return out


def bits(v: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", v))[0]


def dense(s: str) -> gen.CSR:
    return gen.from_dense(np.array([[num(v) for v in r.split(",")] for r in s.split(";")]))


# ------------------------------------------------------------------ oracle --

@pytest.mark.parametrize("case", rows("spec_exdot.txt"), ids=lambda c: c[0])
def test_oracle_exdot_golden(case):
    _, x, y, want, _line = case
    v, f = oracle.exdot(vec(x), vec(y))
    # RANGE may be set (R-9: 2^-1074 lies below the GPU fast pass's exact zone); the value is exact either way
    assert not (f & oracle.F_NONFINITE) and bits(v) == bits(num(want)), (case, v)


@pytest.mark.parametrize("case", rows("spec_dot_sequential.txt"), ids=lambda c: c[0])
def test_oracle_sequential_dot_golden(case):
    _, x, y, want, _line = case
    assert bits(oracle.dot_seq(vec(x), vec(y))) == bits(num(want))


@pytest.mark.parametrize("case", rows("spec_partition.txt"), ids=lambda c: c[0] + "/" + c[1])
def test_partition_golden(case):
    # host-only C-ABI planning routine (no GPU needed)
    import paper_2404_13216_b200 as pb
    n, p, want, _line = int(case[0]), int(case[1]), case[2], case[3]
    b = pb.plan_partition(n, p)
    sizes = np.diff(b)
    assert b[0] == 0 and b[-1] == n and (sizes > 0).all()
    if want.startswith("set:"):
        assert set(sizes.tolist()) <= {int(v) for v in want[4:].split(",")}
    else:
        assert sizes.tolist() == [int(v) for v in want.split(",")]


@pytest.mark.parametrize("case", rows("spec_spmv.txt"), ids=lambda c: c[0])
def test_oracle_spmv_golden(case):
    _, m, x, want, _line = case
    y = oracle.spmv(dense(m), vec(x))
    assert [bits(v) for v in y] == [bits(v) for v in vec(want)]


@pytest.mark.parametrize("case", rows("spec_solver.txt"), ids=lambda c: c[0])
def test_oracle_solver_golden(case):
    name, m, b, x0, want, iters, _line = case
    A = dense(m)
    if name.startswith("bicgstab"):
        st, it, x, _ = oracle.bicgstab(A, vec(b), vec(x0), tol=1e-10, max_iter=10)
        assert st == oracle.CONVERGED
    else:
        O = oracle.PBiCGStab(A, b=vec(b), tol=1e-10, max_iter=10)
        O.run()
        assert O.status == oracle.CONVERGED
        it, x = O.iterations, O.vec("x")
    assert it == int(iters) and [bits(v) for v in x] == [bits(v) for v in vec(want)]


@pytest.mark.parametrize("case", rows("spec_true_residual.txt"), ids=lambda c: c[0])
def test_oracle_true_residual_golden(case):
    _, d, b, x, want, _line = case
    A = gen.from_dense(np.diag(vec(d)))
    r, f = oracle.true_relres(A, vec(b), vec(x))
    assert f == 0 and bits(r) == bits(num(want))


# --------------------------------------------------------------------- GPU --

@pytest.fixture(scope="module")
def pb():
    import torch
    assert torch.cuda.is_available()
    import paper_2404_13216_b200 as pb
    return pb


@pytest.mark.gpu
@pytest.mark.parametrize("case", rows("spec_exdot.txt"), ids=lambda c: c[0])
def test_gpu_exdot_golden(pb, case):
    import torch
    _, x, y, want, _line = case
    v, f = pb.exdot(torch.from_numpy(vec(x)).cuda(), torch.from_numpy(vec(y)).cuda())
    assert not (f & pb.FLAG_NONFINITE) and bits(v) == bits(num(want)), (case, v)  # RANGE: full-range pass, exact


@pytest.mark.gpu
@pytest.mark.parametrize("case", rows("spec_spmv.txt"), ids=lambda c: c[0])
def test_gpu_spmv_golden(pb, case):
    import torch
    _, m, x, want, _line = case
    A = dense(m)
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n)
    y = S.spmv(torch.from_numpy(vec(x)).cuda()).cpu().numpy()
    S.close()
    assert [bits(v) for v in y] == [bits(v) for v in vec(want)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", rows("spec_solver.txt"), ids=lambda c: c[0])
def test_gpu_solver_golden(pb, case):
    import torch
    name, m, b, x0, want, iters, _line = case
    A = dense(m)
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n)
    method = "bicgstab" if name.startswith("bicgstab") else "pbicgstab"
    x, r = S.solve(torch.from_numpy(vec(b)).cuda(), x0=torch.from_numpy(vec(x0)).cuda(), tol=1e-10, max_iter=10,
                   method=method)
    S.close()
    assert r.status == pb.CONVERGED and r.iterations == int(iters)
    assert [bits(v) for v in x.cpu().numpy()] == [bits(v) for v in vec(want)]


@pytest.mark.gpu
@pytest.mark.parametrize("case", rows("spec_true_residual.txt"), ids=lambda c: c[0])
def test_gpu_true_residual_golden(pb, case):
    # max_iter = 0: the solve stops at initialisation, finish() reports
    # NORM(b - A x0) / NORM(b) for the given x0
    import torch
    _, d, b, x, want, _line = case
    A = gen.from_dense(np.diag(vec(d)))
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n)
    _, r = S.solve(torch.from_numpy(vec(b)).cuda(), x0=torch.from_numpy(vec(x)).cuda(), tol=0.0, max_iter=0)
    S.close()
    assert bits(r.relres_true) == bits(num(want))
