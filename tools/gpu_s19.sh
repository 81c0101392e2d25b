O=gpurun_out/s19; mkdir -p $O
L=$PWD/paper_2404_13216_b200
V="$L/libpbicgstab.so $L/libpbicgstab_k3l9.so $L/libpbicgstab_k3l10.so"
timeout 900 python tools/ab_iter.py c3_3d128 400 $V > $O/ab_c3.txt 2>&1
timeout 900 python tools/ab_iter.py c4_rand4m 200 $V > $O/ab_c4.txt 2>&1
