"""Phase times of the fused small-system kernel (debug build, CTA 0):
PBCG_LIB=paper_2404_13216_b200/libpbicgstab_dbg.so python tools/diag_small.py [workload] [K]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
A = gen.make_config(sys.argv[1] if len(sys.argv) > 1 else "c1_2d64")
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=8)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
for dm in ("exact", "plain"):
    S.start(b, tol=0.0, max_iter=K + 20, dot_mode=dm)
    S.iterate(10)
    torch.cuda.synchronize()
    pb.debug_counters(reset=True)
    S.iterate(K)
    torch.cuda.synchronize()
    c = pb.debug_counters(reset=True).astype(np.float64) / K / 1e3
    names = {4: "K2 rows+publish", 5: "barrier A", 6: "round A", 7: "SpMV v", 13: "K3 rows+publish", 14: "barrier B",
             15: "round B + SpMV t"}
    print(dm, "us/iteration:", {v: round(c[k], 2) for k, v in names.items()}, "total", round(sum(c[k] for k in names), 2))
    S.finish(None)
S.close()
