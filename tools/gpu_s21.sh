O=gpurun_out/s21; mkdir -p $O
L=$PWD/paper_2404_13216_b200
V="$L/libpbicgstab.so $L/libpbicgstab_v432.so $L/libpbicgstab_v422.so $L/libpbicgstab_v333.so $L/libpbicgstab_k3v422.so"
WARM=5 timeout 900 python tools/ab_iter.py c5_3d256 20 $V > $O/ab_c5_k20.txt 2>&1
WARM=20 timeout 900 python tools/ab_iter.py c5_3d256 200 $V > $O/ab_c5_k200.txt 2>&1
