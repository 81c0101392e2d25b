O=gpurun_out/s4; mkdir -p $O
L=$PWD/paper_2404_13216_b200
for v in dbg dbg6 dbgold; do
  PBCG_LIB=$L/libpbicgstab_$v.so timeout 600 python tools/diag_spill.py c5_3d256 x > $O/diag_c5_$v.txt 2>&1
  PBCG_LIB=$L/libpbicgstab_$v.so timeout 600 python tools/diag_spill.py c3_3d128 > $O/diag_c3_$v.txt 2>&1
done
timeout 900 python tools/ab_iter.py c5_3d256 200 $L/libpbicgstab_c6.so $L/libpbicgstab_old.so > $O/ab_c5.txt 2>&1
PBCG_LIB=$L/libpbicgstab_c6.so timeout 300 python tools/exdot_bench.py 26 > $O/exdot26_c6.json 2>&1
ls -la $O
