"""Order-1/2 cfg3 latency through bench.latency (used for zero-copy A/B: RTN_ZEROCOPY=0/1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
S = [17] + [512] * 12 + [6]
for order in (1, 2):
    r = bench.latency(torch, S, 12512, 20, steps=300, order=order)
    print(f"order {order}: p50 {r['p50_us']:.1f} p99 {r['p99_us']:.1f} device p50 {r['device_p50_us']:.1f}", flush=True)
