"""Phase timestamps of K2 (debug build): PBCG_LIB=..._dbg.so python tools/diag_ts.py c1_2d64
Prints, per launch, the latest time (over warps) each phase ended, relative to the latest start."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
A = gen.make_config(sys.argv[1])
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=64)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
S.start(b, tol=0.0, max_iter=60)
S.iterate(5); torch.cuda.synchronize()
for rep in range(3):
    pb.debug_counters(reset=True)
    ms = S.profile(1)
    c = pb.debug_counters(reset=True).astype(np.int64)
    t = c[8:13]
    print(f"K2 {ms[0]*1e3:.1f} us; start->tiles {(t[1]-t[0])/1e3:.1f} ->merged {(t[2]-t[1])/1e3:.1f} ->published {(t[3]-t[2])/1e3:.1f} us (end of kernel = max over CTAs)")
