#!/bin/bash
# Register / spill summary of the stream kernels for a set of defines:
#   tools/regs.sh [DEFINE...]   (e.g. PBCG_S_NCW=8)
D=""; for d in "$@"; do D="$D -D$d"; done
NCCL=$(python -c "import sys; sys.path.insert(0,'paper_2404_13216_b200'); import build; print(build.nccl_include())")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false -Xptxas=-v -cubin \
  -I include -I $NCCL $D -o /tmp/regs.cubin paper_2404_13216_b200/csrc/runtime.cu 2>&1 | python3 -c '
import sys, re
cur = None
for l in sys.stdin:
    m = re.search(r"Compiling entry function .(_ZN4pbcg\w+)", l)
    if m:
        n = m.group(1)
        cur = n if re.search(r"k2_stream|k3_stream|exdot_stream", n) else None
        if cur:
            t = re.search(r"(k2_stream|k3_stream|exdot_stream)I(.*)EEEv", n)
            cur = t.group(1) + "<" + ",".join(re.findall(r"L([ib])(\d+)E", t.group(2)) and [v for _, v in re.findall(r"L([ib])(\d+)E", t.group(2))]) + ">"
        continue
    if cur and "spill" in l:
        sp = re.search(r"(\d+) bytes spill stores", l).group(1)
    if cur and "registers" in l:
        print(f"{cur:40s} regs {re.search(r"Used (\d+) registers", l).group(1):>4s} spill {sp}")
        cur = None
'
