set -x
O=gpurun_out/s3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_accumulator.py -x -q > $O/acc.log 2>&1; echo "rc=$?" >> $O/acc.log
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
L=$PWD/paper_2404_13216_b200
V="$L/libpbicgstab.so $L/libpbicgstab_h21.so $L/libpbicgstab_h22.so $L/libpbicgstab_old.so"
timeout 900 python tools/ab_iter.py c5_3d256 200 $V > $O/ab_c5.txt 2>&1
timeout 900 python tools/ab_iter.py c3_3d128 400 $V > $O/ab_c3.txt 2>&1
timeout 900 python tools/ab_iter.py c4_rand4m 200 $V > $O/ab_c4.txt 2>&1
for l in libpbicgstab libpbicgstab_h21 libpbicgstab_h22 libpbicgstab_old; do PBCG_LIB=$L/$l.so timeout 300 python tools/exdot_bench.py 26 > $O/exdot26_$l.json 2>&1; done
ls -la $O
