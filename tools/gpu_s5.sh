O=gpurun_out/s5; mkdir -p $O
L=$PWD/paper_2404_13216_b200
timeout 900 python tools/ab_iter.py c5_3d256 200 $L/libpbicgstab.so $L/libpbicgstab_old.so > $O/ab_c5.txt 2>&1
timeout 900 python tools/ab_iter.py c3_3d128 400 $L/libpbicgstab.so $L/libpbicgstab_old.so > $O/ab_c3.txt 2>&1
timeout 900 python tools/ab_iter.py c4_rand4m 200 $L/libpbicgstab.so $L/libpbicgstab_old.so > $O/ab_c4.txt 2>&1
timeout 300 python tools/exdot_bench.py 26 > $O/exdot26.json 2>&1

