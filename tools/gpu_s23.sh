O=gpurun_out/s23; mkdir -p $O
L=$PWD/paper_2404_13216_b200
V="$L/libpbicgstab.so $L/libpbicgstab_old.so"
timeout 900 python tools/ab_iter.py c1_2d64 2000 $V > $O/ab_c1.txt 2>&1
timeout 900 python tools/ab_iter.py c3_3d128 400 $V > $O/ab_c3.txt 2>&1
WARM=5 timeout 900 python tools/ab_iter.py c5_3d256 20 $V > $O/ab_c5_k20.txt 2>&1
timeout 900 python tools/ab_iter.py c4_rand4m 200 $V > $O/ab_c4.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
