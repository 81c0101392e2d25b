"""Per-CTA phase timeline of one iteration (PBCG_TIMELINE build):
PBCG_LIB=paper_2404_13216_b200/libpbicgstab_tl.so python tools/timeline.py [workload]
Phases: K2/K3 0 entry, 1 after the PDL wait, 2 first tile landed, 3 tiles
done (warp 0), 4 FPEs drained, 5 published, 6 every warp done with its tiles; SpMV 0 entry, 1 after the wait, 2 first
chunk landed, 3 done.  Times in us relative to the earliest release of K2's PDL wait
(chained graphs: python tools/timeline.py c3_3d128 10, the last iteration):
min / median / max over CTAs."""
import sys, os, ctypes
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
L = pb.lib()
L.pbcg_timeline.argtypes = [ctypes.c_void_p, ctypes.c_int32]
A = gen.make_config(sys.argv[1] if len(sys.argv) > 1 else "c3_3d128")
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
CH = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # iterations per graph: the stamps are the last one's
S.start(b, tol=0.0, max_iter=400, poll_every=CH)
S.iterate(20 * CH)
torch.cuda.synchronize()
buf = np.zeros((3, 256, 8), np.uint64)
for rep in range(3):
    L.pbcg_timeline(buf.ctypes.data, 1)
    S.iterate(CH)
    torch.cuda.synchronize()
    L.pbcg_timeline(buf.ctypes.data, 1)
    t = buf.astype(np.int64)
    t0 = t[0, :, 1][t[0, :, 1] > 0].min()  # K2's PDL wait released
    print(f"--- iteration {rep}")
    for kind, nm, nph in ((0, "K2", 7), (1, "SpMV", 4), (2, "K3", 7)):
        for k in range(nph):
            v = t[kind, :, k]
            v = v[v > 0]
            if v.size == 0:
                continue
            v = (v - t0) / 1e3
            print(f"{nm:5s} ph{k}: min {v.min():7.2f} med {np.median(v):7.2f} max {v.max():7.2f}  (n={v.size})")
S.finish(None)
S.close()
# K2: tiles-done time per CTA against its SM id (is the spread systematic?)
t = buf.astype(np.int64)
sm = t[0, :148, 7]
d = (t[0, :148, 3] - t[0, :148, 1]) / 1e3
o = np.argsort(sm)
print("K2 stream time (ph1->ph3) by SM id:")
print(" ".join(f"{int(sm[i])}:{d[i]:.0f}" for i in o))
print("by blockIdx:", " ".join(f"{v:.0f}" for v in d))
