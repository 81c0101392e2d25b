"""Spill statistics with the counter build: PBCG_LIB=.../libpbicgstab_dbg.so python tools/diag_spill.py c5_3d256"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
name = sys.argv[1]
A = gen.make_config(name)
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=512)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
S.start(b, tol=0.0, max_iter=400)
for it in (0, 10, 50, 100, 200):
    cur = S.finish(None).iterations
    if it > cur:
        S.iterate(it - cur)
    torch.cuda.synchronize()
    pb.debug_counters(reset=True)
    ms = S.profile(1)
    c = pb.debug_counters(reset=True)
    print(f"{name} iter {it}: products {7*A.n} c1 {c[1]} ({32*c[1]/(7*A.n):.3%} x32) c2 {c[2]} deposits {c[3]} ({c[3]/(7*A.n):.3%})  ms K2 {ms[0]:.3f} K3 {ms[2]:.3f}")
if len(sys.argv) > 2:
    n = 1 << 24
    for kind, (x, y) in (("well", (gen.uniform(n, 1), gen.uniform(n, 2))), ("ill", gen.ill_pair(n, seed=3))):
        pb.debug_counters(reset=True)
        pb.exdot(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda())
        c = pb.debug_counters(reset=True)
        print(f"exdot {kind}: n {n} c1 {c[1]} ({32*c[1]/n:.3%} x32) c2 {c[2]} deposits {c[3]} ({c[3]/n:.3%})")
