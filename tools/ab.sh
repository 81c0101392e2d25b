#!/bin/bash
# A/B the library variants on one workload: tools/ab.sh WORKLOAD STEPS variant...
W=$1; K=$2; shift 2
for v in "$@"; do
  if [ "$v" = "main" ]; then L=$PWD/paper_2404_13216_b200/libpbicgstab.so; else L=$PWD/paper_2404_13216_b200/libpbicgstab_$v.so; fi
  PBCG_LIB=$L timeout 300 python bench.py --workload $W --no-e2e --no-extras --steps $K > gpurun_out/ab_${W}_$v.json 2> gpurun_out/ab_${W}_$v.err
done
