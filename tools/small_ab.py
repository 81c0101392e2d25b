"""Fused small-system kernel vs the six-kernel path (PBCG_SMALL=0) on
matrices around the size threshold: python tools/small_ab.py [K]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, paper_2404_13216_b200 as pb
K = int(sys.argv[1]) if len(sys.argv) > 1 else 300
mats = {"c1": lambda: gen.make_config("c1_2d64"), "3d24": lambda: gen.stencil(3, 24, 100.0),
        "2d128": lambda: gen.stencil(2, 128, 10.0), "3d32": lambda: gen.stencil(3, 32, 100.0),
        "3d40": lambda: gen.stencil(3, 40, 100.0), "3d50": lambda: gen.stencil(3, 50, 100.0),
        "rand32k": lambda: gen.random_banded(32_768, seed=3, band=2000),
        "rand128k": lambda: gen.random_banded(131_072, seed=3, band=5000)}
for name, mk in mats.items():
    A = mk()
    row = {"name": name, "n": A.n}
    for env in ("1", "0"):
        os.environ["PBCG_SMALL"] = env
        S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=8)
        b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
        S.start(b, tol=0.0, max_iter=K + 20)
        mode = S.exec_mode()
        S.iterate(10)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(S.stream)
        S.iterate(K)
        e1.record(S.stream)
        torch.cuda.synchronize()
        r = S.finish(None)
        row[f"mode{mode}"] = round(K / (e0.elapsed_time(e1) * 1e-3))
        S.close()
    print(json.dumps(row), flush=True)
