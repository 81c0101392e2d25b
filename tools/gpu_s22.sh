O=gpurun_out/s22; mkdir -p $O
L=$PWD/paper_2404_13216_b200
V="$L/libpbicgstab.so $L/libpbicgstab_f2s.so"
for l in libpbicgstab libpbicgstab_f2s; do PBCG_LIB=$L/$l.so timeout 300 python tools/exdot_bench.py 26 > $O/exdot26_$l.json 2>&1; done
WARM=5 timeout 900 python tools/ab_iter.py c5_3d256 20 $V > $O/ab_c5_k20.txt 2>&1
timeout 900 python tools/ab_iter.py c3_3d128 400 $V > $O/ab_c3.txt 2>&1
timeout 900 python tools/ab_iter.py c4_rand4m 200 $V > $O/ab_c4.txt 2>&1
PBCG_LIB=$L/libpbicgstab_f2s.so timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_f2s.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_f2s.log
