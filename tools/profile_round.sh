#!/bin/bash
# End-of-round measurement pass on one GPU (run under gpurun):
#   bench lines for every workload + the reference (oracle) arm, the ncu launch
#   list of the C5 bench, and one `ncu --set full` capture of the hot kernels
#   (C5 iteration, C4 SELL-V SpMV, C1 cluster kernel, EXDOT 2^26 WELL and ILL).
# Output: gpurun_out/$1/ (default r01d).  Each ncu pass runs after the same
# command has exited 0 without ncu.
OUT=gpurun_out/${1:-r03}
mkdir -p $OUT
for w in c5_3d256 c4_rand4m c3_3d128 c1_2d64; do
  timeout 900 python bench.py --workload $w > $OUT/bench_$w.json 2> $OUT/bench_$w.err || echo "bench $w failed"
done
# the driver's own command (K = 20, W = 5), both arms
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_c5_k20_w5.json 2> $OUT/bench_c5_k20_w5.err || echo "bench k20 failed"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2> $OUT/bench_reference.err || echo "reference failed"
# launch list (cold, serialised; shares only)
timeout 600 python bench.py --steps 20 --warmup 3 --no-extras --no-e2e > $OUT/b_nx.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_c5.csv \
  python bench.py --steps 20 --warmup 3 --no-extras --no-e2e > $OUT/ncu_launch.log 2>&1 || echo "launch list failed"
# full captures: C5 iteration kernels at iteration ~10
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k2_stream|k3_stream|spmv_sellp_kernel|finalize_kernel" --launch-skip 60 --launch-count 6 \
  -o $OUT/ncu_full_c5 python bench.py --steps 20 --warmup 3 --no-extras --no-e2e > $OUT/ncu_full_c5.log 2>&1 || echo "c5 full failed"
# C3 iteration kernels (lean K2/K3, SELL-P SpMV) at iteration ~10
timeout 600 python bench.py --workload c3_3d128 --steps 20 --warmup 3 --no-extras --no-e2e > $OUT/b_c3_nx.json 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k2_stream|k3_stream|spmv_sellp_kernel|finalize_kernel" --launch-skip 60 --launch-count 6 \
  -o $OUT/ncu_full_c3 python bench.py --workload c3_3d128 --steps 20 --warmup 3 --no-extras --no-e2e > $OUT/ncu_full_c3.log 2>&1 || echo "c3 full failed"
# C4 SELL-V SpMV
timeout 300 python tools/spmv_bench.py c4_rand4m 5 > $OUT/spmv_c4.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:spmv_sellv -s 3 -c 1 \
  -o $OUT/ncu_full_c4_sellv python tools/spmv_bench.py c4_rand4m 5 > $OUT/ncu_full_c4.log 2>&1 || echo "c4 full failed"
# C1 cluster kernel (the timed launch: 200 iterations)
timeout 300 python bench.py --workload c1_2d64 --steps 200 --warmup 10 --no-extras --no-e2e > $OUT/b_c1_nx.json 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"pbcg_cluster|pbcg_small" -s 1 -c 1 \
  -o $OUT/ncu_full_c1_cluster python bench.py --workload c1_2d64 --steps 200 --warmup 10 --no-extras --no-e2e \
  > $OUT/ncu_full_c1.log 2>&1 || echo "c1 full failed"
# EXDOT stream kernel at 2^26: launch 0 = WELL, launch 13 = ILL (3 warm-ups + 10 timed per case)
timeout 300 python tools/exdot_bench.py 26 > $OUT/exdot26.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exdot_stream -s 0 -c 1 \
  -o $OUT/ncu_full_exdot_well python tools/exdot_bench.py 26 > $OUT/ncu_full_exdot_well.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exdot_stream -s 13 -c 1 \
  -o $OUT/ncu_full_exdot_ill python tools/exdot_bench.py 26 > $OUT/ncu_full_exdot_ill.log 2>&1 || echo "exdot full failed"

# summaries on the box (the .ncu-rep files are too large to bring back)
for r in $OUT/*.ncu-rep; do python tools/ncu_summary.py full $r > ${r%.ncu-rep}.jsonl 2>&1; done
python tools/ncu_summary.py launches $OUT/launches_c5.csv > $OUT/launches_c5.md 2>&1
rm -f $OUT/*.ncu-rep
ls -la $OUT
