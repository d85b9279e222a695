"""cfg1/cfg2/cfg3 (order 1 and 2) latency, one line each (bench.latency)."""
import sys, torch
sys.path.insert(0, ".")
import bench
S = [17] + [512] * 12 + [6]
for name, sizes, seed, k, order, prec, act in (("cfg3", S, 12512, 20, 1, 0, "silu"), ("cfg3 order2", S, 12512, 20, 2, 0, "silu"),
                                               ("cfg3 bf16", S, 12512, 20, 1, 3, "silu"),
                                               ("cfg2", [17] + [256] * 5 + [6], 5256, 20, 1, 0, "silu"),
                                               ("cfg1", [17, 64, 64, 6], 2064, 10, 1, 0, "tanh")):
    r = bench.latency(torch, sizes, seed, k, steps=500, order=order, precision=prec, act=act)
    print(f"{name}: p50 {r['p50_us']:.1f} p99 {r['p99_us']:.1f} device p50 {r['device_p50_us']:.1f}", flush=True)
