"""Runs bench.blocks_bench alone (GPU)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
t0 = time.time()
r = bench.blocks_bench(torch, json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"])
print(json.dumps(r, indent=1))
print("wall", time.time() - t0)
