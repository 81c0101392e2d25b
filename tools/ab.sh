#!/bin/bash
# A/B the library variants on one workload: tools/ab.sh WORKLOAD STEPS variant...
# variant: main | <name> (libpbicgstab_<name>.so) | env:VAR=VALUE (main lib + env)
W=$1; K=$2; shift 2
for v in "$@"; do
  L=$PWD/paper_2404_13216_b200/libpbicgstab.so; E=""
  case "$v" in
    main) ;;
    env:*) E="${v#env:}";;
    *) L=$PWD/paper_2404_13216_b200/libpbicgstab_$v.so;;
  esac
  tag=$(echo "$v" | tr ':=' '__')
  env $E PBCG_LIB=$L timeout 300 python bench.py --workload $W --no-e2e --no-extras --steps $K > gpurun_out/ab_${W}_$tag.json 2> gpurun_out/ab_${W}_$tag.err
done
