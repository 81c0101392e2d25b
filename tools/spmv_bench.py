"""SpMV-only timing for A/B runs: python tools/spmv_bench.py c5_3d256 [K]
Times K pbicgstab_spmv calls (each = D2D copy of x into the padded buffer +
the SpMV kernel) with CUDA events and subtracts the same number of plain
D2D copies of x."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, gen, paper_2404_13216_b200 as pb
name = sys.argv[1]; K = int(sys.argv[2]) if len(sys.argv) > 2 else 50
if name.startswith("c4band"):  # C4 with another band: c4band1000
    A = gen.random_banded(1 << 22, seed=42, band=int(name[6:]))
else:
    A = gen.make_config(name)
S = pb.Solver(A.row_ptr, A.col, A.val, A.n)
x = torch.from_numpy(gen.uniform(A.n, 5)).cuda()
for _ in range(3):
    S.spmv(x)
torch.cuda.synchronize()
e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
st = torch.cuda.current_stream()
e0.record()
for _ in range(K):
    S.spmv(x)
e1.record()
buf = torch.empty_like(x)
for _ in range(K):
    buf.copy_(x)
e2.record()
torch.cuda.synchronize()
t_all = e0.elapsed_time(e1) / K * 1e3
t_cp = e1.elapsed_time(e2) / K * 1e3
f = S.spmv_format()
print(json.dumps({"workload": name, "spmv_us": t_all - t_cp, "call_us": t_all, "copy_us": t_cp,
                  "GBps_fmt": f["bytes_per_spmv"] / ((t_all - t_cp) * 1e-6) / 1e9, "fmt": f,
                  "env": {k: v for k, v in os.environ.items() if k.startswith("PBCG")}}))
