set -x
mkdir -p gpurun_out/s1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/s1/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/s1/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/s1/bench_c5.json 2> gpurun_out/s1/bench_c5.err
timeout 600 python bench.py --workload c3_3d128 > gpurun_out/s1/bench_c3.json 2> gpurun_out/s1/bench_c3.err
timeout 300 python tools/exdot_bench.py 26 > gpurun_out/s1/exdot26.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exdot_stream -s 0 -c 1 -o gpurun_out/s1/ncu_full_exdot_well python tools/exdot_bench.py 26 > gpurun_out/s1/ncu_exdot_well.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:exdot_stream -s 13 -c 1 -o gpurun_out/s1/ncu_full_exdot_ill python tools/exdot_bench.py 26 > gpurun_out/s1/ncu_exdot_ill.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k2_stream|k3_stream" --launch-skip 20 --launch-count 2 -o gpurun_out/s1/ncu_full_c5_k23 python bench.py --steps 20 --warmup 3 --no-extras --no-e2e > gpurun_out/s1/ncu_c5.log 2>&1
ls -la gpurun_out/s1
