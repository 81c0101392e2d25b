#!/bin/bash
# compute-sanitizer passes over the small-system and solver paths (run under gpurun):
#   tools/sanitize.sh [OUTDIR]   -> OUTDIR/{memcheck,racecheck,synccheck,initcheck}_*.txt
# memcheck: out-of-bounds / misaligned accesses (global, shared, TMA bulk copies); racecheck: shared-memory
# hazards; synccheck: barrier misuse; initcheck: reads of uninitialised global memory.  Small inputs only:
# the tools slow kernels down 10-100x.
O=${1:-gpurun_out/sanitize}; mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
SMOKE='import __graft_entry__ as g; g.smoke()'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python -c "$SMOKE" > $O/${tool}_smoke.txt 2>&1
  echo "rc=$?" >> $O/${tool}_smoke.txt
done
# the six-kernel path on a mid-size stencil (TMA rings, PDL, SELL-P) and the SELL-V path, memcheck only
cat > /tmp/san_mid.py <<'P'
import sys, os; sys.path.insert(0, os.getcwd())
import numpy as np, torch, gen, paper_2404_13216_b200 as pb
for A in (gen.stencil(3, 48, 100.0), gen.random_banded(70000, seed=5), gen.stencil(2, 64, 10.0)):
    S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=64)
    b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
    r = S.solve(b, tol=0.0, max_iter=6)
    print(A.name, A.n, "exec_mode", S.exec_mode(), S.spmv_format(), r.status, r.iterations, r.relres_recursive, r.relres_true)
    x, y = torch.from_numpy(gen.uniform(300001, 1)).cuda(), torch.from_numpy(gen.uniform(300001, 2)).cuda()
    print("exdot", pb.exdot(x, y))
P
for tool in memcheck racecheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 python /tmp/san_mid.py > $O/${tool}_mid.txt 2>&1
  echo "rc=$?" >> $O/${tool}_mid.txt
done
