"""Convergence diagnostics on the GPU: recursive relres history, true relres,
iterations, for a BASELINE config (prints a compact table)."""
import sys, os, json, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import gen, paper_2404_13216_b200 as pb
name = sys.argv[1]; max_iter = int(sys.argv[2]) if len(sys.argv) > 2 else 3000
A = gen.make_config(name)
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=max_iter + 1)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
t = time.time()
x, r = S.solve(b, tol=1e-10, max_iter=max_iter, poll_every=32)
torch.cuda.synchronize()
el = time.time() - t
H = S.history()
rel = H[:, 8]
step = max(1, len(rel) // 40)
print(json.dumps({"config": name, "status": r.status_name, "iterations": r.iterations, "relres": r.relres_recursive,
                  "relres_true": r.relres_true, "loop_s": r.loop_seconds, "wall_s": el,
                  "err_vs_ones": float((x - 1).abs().max()) if A.rhs != "given" else None}))
for i in range(0, len(rel), step):
    print(i, "%.3e" % rel[i], "omega=%.3e alpha=%.3e" % (H[i, 4], H[i, 10]))
