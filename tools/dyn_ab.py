"""A/B of an environment switch on the iteration rate, interleaved in one
process: python tools/dyn_ab.py VAR workload [K] (VAR=1 vs VAR=0)"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
var = sys.argv[1]
A = gen.make_config(sys.argv[2] if len(sys.argv) > 2 else "c3_3d128")
K = int(sys.argv[3]) if len(sys.argv) > 3 else 100
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
res = {"1": [], "0": []}
for rep in range(4):
    for v in ("1", "0"):
        os.environ[var] = v
        S.start(b, tol=0.0, max_iter=K + 40, poll_every=10)  # start() captures the graph with the switch
        S.iterate(20)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(S.stream); S.iterate(K); e1.record(S.stream); torch.cuda.synchronize()
        S.finish(None)
        res[v].append(K / (e0.elapsed_time(e1) * 1e-3))
for v in ("1", "0"):
    print(f"{var}={v}: {np.median(res[v]):9.1f} iter/s  {[round(x) for x in res[v]]}")
S.close()
