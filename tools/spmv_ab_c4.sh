# C4 SpMV A/B of SELL-V library variants (tools/spmv_bench.py), interleaved
L=$PWD/paper_2404_13216_b200
for rep in 1 2; do for v in "" "$@"; do
  echo -n "lib$v: "; PBCG_LIB=$L/libpbicgstab$v.so python tools/spmv_bench.py c4_rand4m 20 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['spmv_us'],1), round(d['GBps_fmt']))"
done; done
