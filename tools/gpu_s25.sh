O=gpurun_out/s25; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 600 python tools/e2e_breakdown.py c5_3d256 20 > $O/e2e_c5_k20.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > $O/bench_c5_k20.json 2> $O/bench_c5_k20.err
