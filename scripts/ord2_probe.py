"""cfg3 order-2 latency vs the order-2 tile height (RTN_ORD2_NTC), one setting per process:
  python scripts/ord2_probe.py <tf32|3xtf32|bf16|bf16x3> ; RTN_ORD2_NTC=40 python scripts/ord2_probe.py tf32"""
import os, sys, torch
sys.path.insert(0, ".")
import bench
from paper_2203_07747_b200._lib import PRECISIONS
a = sys.argv[1] if len(sys.argv) > 1 else "tf32"
prec = PRECISIONS[a] if a in PRECISIONS else int(a)  # a name or the rtn_precision value
k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
r = bench.latency(torch, [17] + [512] * 12 + [6], 12512, k, steps=300, order=2, precision=prec)
print(f"ntc={os.environ.get('RTN_ORD2_NTC', 'default')} prec={prec} K={k}: p50 {r['p50_us']:.1f} p99 {r['p99_us']:.1f} "
      f"device p50 {r['device_p50_us']:.1f}", flush=True)
