"""cfg3 latency per precision mode (bench.latency); run with and without RTN_QUAD=0."""
import sys, torch
sys.path.insert(0, ".")
import bench
S = [17] + [512] * 12 + [6]
for prec, name in ((0, "tf32"), (1, "3xtf32"), (2, "bf16x3")):
    r = bench.latency(torch, S, 12512, 20, steps=300, precision=prec)
    print(f"{name} cfg3 latency: p50 {r['p50_us']:.1f} p99 {r['p99_us']:.1f} device p50 {r['device_p50_us']:.1f}", flush=True)
