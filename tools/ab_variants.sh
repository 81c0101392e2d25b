#!/bin/bash
# A/B of library variants on the GPU box (run under gpurun), the procedure behind every "measured and rejected"
# line of DESIGN.md: build each variant here first,
#   python paper_2404_13216_b200/build.py --variant NAME DEFINE...      (e.g. --variant lean3 PBCG_LEAN_NH=3)
# then:  tools/ab_variants.sh WORKLOAD K NAME...   (main = the default library)
# Prints iter/s per variant, interleaved over 3 repetitions (tools/ab_iter.py; WARM= and PRECOND= pass through).
W=$1; K=$2; shift 2
L=$PWD/paper_2404_13216_b200
V=""
for n in "$@"; do
  if [ "$n" = main ]; then V="$V $L/libpbicgstab.so"; else V="$V $L/libpbicgstab_$n.so"; fi
done
timeout 900 python tools/ab_iter.py "$W" "$K" $V
