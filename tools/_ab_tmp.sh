mkdir -p gpurun_out/ab
tools/ab_variants.sh c3_3d128 200 main drain2 > gpurun_out/ab/drain2.txt 2>&1
WARM=5 tools/ab_variants.sh c5_3d256 20 main drain2 >> gpurun_out/ab/drain2.txt 2>&1
tools/ab_variants.sh c4_rand4m 100 main drain2 >> gpurun_out/ab/drain2.txt 2>&1
for v in "" _drain2 "" _drain2; do PBCG_LIB=$PWD/paper_2404_13216_b200/libpbicgstab$v.so python tools/exdot_bench.py 26; done >> gpurun_out/ab/drain2.txt 2>&1
PBCG_LIB=$PWD/paper_2404_13216_b200/libpbicgstab_drain2.so timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/ab/pytest_drain2.txt 2>&1
