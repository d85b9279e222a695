"""Fused-cycle latency (bench.cycle_latency: rtn_cycle_qp through the C-ABI, cfg3) for A/B runs:
  RTN_PDL=0 / RTN_BLK_HS=0 python scripts/cycle_abi_probe.py"""
import os, sys
sys.path.insert(0, ".")
import torch
import bench
tag = " ".join(f"{k}={os.environ[k]}" for k in ("RTN_PDL", "RTN_BLK_HS") if k in os.environ) or "default"
for order in (1, 2):
    r = bench.cycle_latency(torch, order, steps=500)
    print(f"{tag}: cycle order {order} p50 {r['p50_us']:.1f} p99 {r['p99_us']:.1f}", flush=True)
