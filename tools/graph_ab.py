"""Timed K iterations with CUDA graphs vs direct launches (same data)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, paper_2404_13216_b200 as pb
name = sys.argv[1]; K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
A = gen.make_config(name)
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
for mode, chunk in (("graph16", 16), ("direct", 1 << 30), ("graph4", 4), ("graph64", 64), ("direct", 1 << 30), ("graph16", 16)):
    pb.lib().pbcg_set_chunk(chunk)
    S.start(b, tol=0.0, max_iter=K + 20)
    S.iterate(10); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(S.stream); S.iterate(K); e1.record(S.stream); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    prof = S.profile(20)
    print(f"{name} {mode:8s}: {ms/K*1e3:8.1f} us/iter  (profiled kernel sum over next 20: {prof.sum()/20*1e3:8.1f} us)")
    S.finish(None)
