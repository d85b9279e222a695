"""cfg3 order-2 latency vs the order-2 tile height (RTN_ORD2_NTC), one setting per process:
  python scripts/ord2_probe.py <precision> ; RTN_ORD2_NTC=40 python scripts/ord2_probe.py 0"""
import os, sys, torch
sys.path.insert(0, ".")
import bench
prec = int(sys.argv[1]) if len(sys.argv) > 1 else 0
k = int(sys.argv[2]) if len(sys.argv) > 2 else 20
r = bench.latency(torch, [17] + [512] * 12 + [6], 12512, k, steps=300, order=2, precision=prec)
print(f"ntc={os.environ.get('RTN_ORD2_NTC', 'default')} prec={prec} K={k}: p50 {r['p50_us']:.1f} p99 {r['p99_us']:.1f} "
      f"device p50 {r['device_p50_us']:.1f}", flush=True)
