O=gpurun_out/s10; mkdir -p $O
L=$PWD/paper_2404_13216_b200
PBCG_LIB=$L/libpbicgstab_tl.so timeout 300 python tools/timeline.py c3_3d128 10 > $O/tl_c3.txt 2>&1
PBCG_LIB=$L/libpbicgstab_tl1.so timeout 300 python tools/timeline.py c3_3d128 10 > $O/tl1_c3.txt 2>&1
