import sys, os
sys.path.insert(0, "/root/repo")
import torch, gen, paper_2404_13216_b200 as pb
A = gen.make_config(sys.argv[1])
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
b = S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
for mode in ("exact", "plain"):
    S.start(b, tol=0.0, max_iter=300, dot_mode=mode)
    S.iterate(10)
    ms = S.profile(100)
    S.finish(None)
    print(mode, " ".join(f"{n} {v*10:.1f}" for n, v in zip(["k2","finA","spmv","k3","finB","spmv"], ms)))
