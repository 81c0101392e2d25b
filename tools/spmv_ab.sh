#!/bin/bash
# SpMV-only A/B: tools/spmv_ab.sh WORKLOAD variant...   (variant: main | <lib name> | env:VAR=VAL[,VAR=VAL])
W=$1; shift
for v in "$@"; do
  L=$PWD/paper_2404_13216_b200/libpbicgstab.so; E=""
  case "$v" in
    main) ;;
    env:*) E="${v#env:}"; E="${E//,/ }";;
    *) L=$PWD/paper_2404_13216_b200/libpbicgstab_$v.so;;
  esac
  echo -n "$v "; env $E PBCG_LIB=$L timeout 300 python tools/spmv_bench.py $W 40 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(f\"spmv {d['spmv_us']:.1f} us  {d['GBps_fmt']:.0f} GB/s(fmt)  explicit {d['fmt']['explicit_cols']}\")" 2>&1
done
