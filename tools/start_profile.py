"""Kernel / copy timeline of pbicgstab_start with a pinned host b (torch.profiler, CUPTI):
python tools/start_profile.py [workload] [finish]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, paper_2404_13216_b200 as pb
from torch.profiler import profile, ProfilerActivity
A = gen.make_config(sys.argv[1] if len(sys.argv) > 1 else "c5_3d256")
S = pb.Solver(A.row_ptr, A.col, A.val, A.n, history_capacity=16)
b = torch.from_numpy(A.b).cuda() if A.rhs == "given" else S.spmv(torch.ones(A.n, dtype=torch.float64, device="cuda"))
bh = torch.empty(A.n, dtype=torch.float64, pin_memory=True); bh.copy_(b.cpu())
for _ in range(2):
    S.start(bh, x0=None, tol=1e-10, max_iter=20); torch.cuda.synchronize()
xh = torch.empty(A.n, dtype=torch.float64, pin_memory=True)
with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    S.start(bh, x0=None, tol=1e-10, max_iter=20)
    torch.cuda.synchronize()
    if len(sys.argv) > 2:  # ... and finish (true residual + copy-out of x)
        S.finish(xh)
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
t0 = min(e.time_range.start for e in ev)
for e in sorted(ev, key=lambda e: e.time_range.start):
    print(f"{(e.time_range.start - t0):9.1f} {(e.time_range.end - t0):9.1f} {e.time_range.end - e.time_range.start:8.1f} us  {e.name[:90]}")
cpu = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CPU]
print("host span:", (max(e.time_range.end for e in cpu) - min(e.time_range.start for e in cpu)), "us")
