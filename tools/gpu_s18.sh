O=gpurun_out/s18; mkdir -p $O
L=$PWD/paper_2404_13216_b200
V="$L/libpbicgstab.so $L/libpbicgstab_lean3.so"
timeout 900 python tools/ab_iter.py c3_3d128 400 $V > $O/ab_c3.txt 2>&1
timeout 900 python tools/ab_iter.py c4_rand4m 200 $V > $O/ab_c4.txt 2>&1
timeout 600 python bench.py --workload c3_3d128 --no-extras > $O/bench_c3.json 2> $O/bench_c3.err
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
