"""Iteration rate of library variants, interleaved, each in its own process:
[PRECOND=bjacobi2_pipe] [WARM=20] python tools/ab_iter.py workload K lib1.so lib2.so ...  (prints iter/s per rep)"""
import sys, os, subprocess, json
w, K, libs = sys.argv[1], sys.argv[2], sys.argv[3:]
code = f"""
import sys, os; sys.path.insert(0, {os.getcwd()!r})
import torch, gen, paper_2404_13216_b200 as pb
A = gen.make_config({w!r}); K = {K}
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16, precond=os.environ.get("PRECOND", "none"))
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
S.start(b, tol=0.0, max_iter=K + 40, poll_every=10); S.iterate({int(os.environ.get("WARM", "20"))}); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(S.stream); S.iterate(K); e1.record(S.stream); torch.cuda.synchronize()
print(K / (e0.elapsed_time(e1) * 1e-3))
"""
res = {l: [] for l in libs}
for rep in range(3):
    for l in libs:
        out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PBCG_LIB=l), capture_output=True, text=True)
        res[l].append(float(out.stdout.strip().splitlines()[-1]))
for l in libs:
    print(f"{w} {os.path.basename(l):28s} {sorted(res[l])[1]:9.1f} iter/s  {[round(x) for x in res[l]]}")
