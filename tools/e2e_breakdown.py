"""Where the end-to-end solve time goes (host buffers): python tools/e2e_breakdown.py [workload] [iters]"""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
A = gen.make_config(sys.argv[1] if len(sys.argv) > 1 else "c5_3d256")
K = int(sys.argv[2]) if len(sys.argv) > 2 else 200
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
bh = torch.empty(A.n, dtype=torch.float64, pin_memory=True); bh.copy_(b.cpu())
xh = torch.zeros(A.n, dtype=torch.float64, pin_memory=True)
st = S.stream
for rep in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    w0 = time.time()
    ev[0].record(st)
    S.start(bh, x0=None, tol=1e-10, max_iter=K)
    ev[1].record(st)
    S.iterate(K)
    ev[2].record(st)
    r = S.finish(xh)
    ev[3].record(st)
    torch.cuda.synchronize()
    w1 = time.time()
    t = [ev[0].elapsed_time(ev[i]) for i in range(1, 4)]
    print(f"start {t[0]:.2f} ms, iterate({K}) {t[1]-t[0]:.2f} ms, finish {t[2]-t[1]:.2f} ms, total {t[2]:.2f} ms, wall {1e3*(w1-w0):.2f} ms")
    # the same through pbicgstab_solve (polls every 16)
    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    f0.record(st)
    x, r = S.solve(bh, x0=None, out=xh, tol=1e-10, max_iter=K, poll_every=16)  # as bench.py's e2e
    f1.record(st)
    torch.cuda.synchronize()
    print(f"solve {f0.elapsed_time(f1):.2f} ms ({r.iterations} iterations)")
# raw copies for reference
d = torch.empty(A.n, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
c0, c1, c2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
c0.record(); d.copy_(bh, non_blocking=True); c1.record(); xh.copy_(d, non_blocking=True); c2.record(); torch.cuda.synchronize()
print(f"H2D {c0.elapsed_time(c1):.2f} ms, D2H {c1.elapsed_time(c2):.2f} ms for {A.n*8/1e6:.0f} MB each")
S.close()
