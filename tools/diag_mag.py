"""Magnitude structure of the K2 products on a config at a few iterations:
per 64-row warp group, the spread (max-min) of log2|product| for (q,y)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
name = sys.argv[1]
A = gen.make_config(name)
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=512)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
S.start(b, tol=0.0, max_iter=400)
done = 0
for it in (1, 10, 50, 200):
    S.iterate(it - done); done = it
    q, y, rh, s, z = (S.vec(k) for k in ("q", "y", "rh", "s", "z"))
    for nm, prod in (("qy", q * y), ("yy", y * y), ("rs", rh * s), ("rz", rh * z)):
        e = np.log2(np.abs(prod[prod != 0])) if (prod != 0).any() else np.array([0.0])
        nz = prod != 0
        g = np.where(nz, np.log2(np.abs(np.where(nz, prod, 1.0))), np.nan).reshape(-1, 64)
        spread = np.nanmax(g, 1) - np.nanmin(g, 1)
        spread = spread[np.isfinite(spread)]
        print(f"it {it} {nm}: zeros {1-nz.mean():.3f} log2 range [{e.min():.0f},{e.max():.0f}] pct(1,50,99)="
              f"{np.percentile(e,1):.0f},{np.percentile(e,50):.0f},{np.percentile(e,99):.0f}  warp-spread median {np.median(spread):.0f} p90 {np.percentile(spread,90):.0f}")
