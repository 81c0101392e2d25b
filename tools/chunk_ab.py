"""Iteration rate vs CUDA-graph chunk length: python tools/chunk_ab.py [workload] [K]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, paper_2404_13216_b200 as pb
A = gen.make_config(sys.argv[1] if len(sys.argv) > 1 else "c3_3d128")
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
for rep in range(2):
    for chunk in (8, 16, 32, 64, K):
        S.start(b, tol=0.0, max_iter=K + 40, poll_every=chunk)
        S.iterate(10)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(S.stream)
        S.iterate(K)
        e1.record(S.stream)
        torch.cuda.synchronize()
        S.finish(None)
        print(f"chunk {chunk:4d}: {K / (e0.elapsed_time(e1) * 1e-3):9.1f} iter/s")
S.close()
