import sys; sys.path.insert(0, ".")
import torch, bench
print(bench.cycle_latency(torch, 2, steps=20)["p50_us"])
