O=gpurun_out/s15; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_solver.py -x -q -k "zero_start or x0_zero" > $O/zs.log 2>&1; echo "rc=$?" >> $O/zs.log
timeout 600 python tools/e2e_breakdown.py c5_3d256 20 > $O/e2e_c5_k20.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > $O/bench_c5_k20.json 2> $O/bench_c5_k20.err
timeout 600 python bench.py --steps 20 --warmup 5 --workload c3_3d128 --no-extras > $O/bench_c3_k20.json 2> $O/bench_c3_k20.err
