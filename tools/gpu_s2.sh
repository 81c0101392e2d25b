set -x
O=gpurun_out/s2; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_bins.py -x -q > $O/bins.log 2>&1; echo "rc=$?" >> $O/bins.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
L=$PWD/paper_2404_13216_b200
timeout 900 python tools/ab_iter.py c5_3d256 200 $L/libpbicgstab.so $L/libpbicgstab_fpe.so > $O/ab_c5.txt 2>&1
timeout 900 python tools/ab_iter.py c3_3d128 400 $L/libpbicgstab.so $L/libpbicgstab_fpe.so > $O/ab_c3.txt 2>&1
timeout 900 python tools/ab_iter.py c4_rand4m 200 $L/libpbicgstab.so $L/libpbicgstab_fpe.so > $O/ab_c4.txt 2>&1
for l in libpbicgstab libpbicgstab_fpe; do PBCG_LIB=$L/$l.so timeout 300 python tools/exdot_bench.py 26 > $O/exdot26_$l.json 2>&1; done
PBCG_LIB=$L/libpbicgstab.so timeout 600 python bench.py --steps 200 --warmup 10 --no-extras > $O/bench_c5.json 2> $O/bench_c5.err
ls -la $O
