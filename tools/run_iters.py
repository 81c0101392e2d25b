"""Run a short p-BiCGStab on a BASELINE config (for ncu captures):
python tools/run_iters.py c5_3d256 12"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, paper_2404_13216_b200 as pb
name = sys.argv[1]; k = int(sys.argv[2]) if len(sys.argv) > 2 else 12
A = gen.make_config(name)
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=64)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
S.start(b, tol=0.0, max_iter=k + 4)
S.iterate(k)
r = S.finish(None)
print("iterations", r.iterations, "status", r.status_name)
if len(sys.argv) > 3:  # also the standalone exdot (WELL, ILL)
    n = 1 << 24
    for x, y in ((gen.uniform(n, 1), gen.uniform(n, 2)), gen.ill_pair(n, seed=3)):
        print("exdot", pb.exdot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()))
