"""Per-kernel fixed cost: serialised per-launch times (pbcg_profile_iterations)
and the graph-replayed iteration time over 3D stencils of growing size; a
linear fit time = a + b n per kernel gives the fixed cost a.
python tools/fixed_cost.py [N ...]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
Ns = [int(v) for v in sys.argv[1:]] or [96, 128, 160, 192]
rows = []
for N in Ns:
    A = gen.stencil(3, N, 100.0)
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
    b = S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
    K = 100
    S.start(b, tol=0.0, max_iter=3 * K + 40, poll_every=10)
    S.iterate(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(S.stream); S.iterate(K); e1.record(S.stream); torch.cuda.synchronize()
    it_us = e0.elapsed_time(e1) / K * 1e3
    ms = S.profile(K) / K * 1e3
    S.finish(None)
    S.close()
    rows.append([A.n, it_us] + list(ms))
    print(f"N={N} n={A.n}: iteration {it_us:.1f} us; K2 {ms[0]:.1f} finA {ms[1]:.1f} SpMV {ms[2]:.1f} K3 {ms[3]:.1f} finB {ms[4]:.1f} SpMV {ms[5]:.1f}", flush=True)
R = np.array(rows)
for j, nm in enumerate(["iteration", "K2", "finA", "SpMVz", "K3", "finB", "SpMVw"]):
    b, a = np.polyfit(R[:, 0], R[:, 1 + j], 1)
    print(f"{nm:10s} fixed {a:7.2f} us, {b * 1e6:7.3f} us per 1M rows")
