"""EXDOT-only timing for A/B runs (bench.py's microbenchmark): python tools/exdot_bench.py [log2n]"""
import sys, os, json, types
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
n = int(sys.argv[1]) if len(sys.argv) > 1 else 26
r = bench.exdot_microbench(types.SimpleNamespace(dot_log2=n), 6554.9)[f"2^{n}"]
print(json.dumps({k: {"exdot_GBps": round(v["exdot"]["GBps"]), "plain": round(v["plain_dot"]["GBps"]),
                      "torch": round(v["torch_dot"]["GBps"]), "flags": v["flags"]} for k, v in r.items() if k != "n"}))
