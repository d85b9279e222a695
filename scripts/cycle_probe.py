"""Latency-mode fused cycle (cfg3: 12x512, N=20): host p50, for ncu launch lists."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import bench
from paper_2203_07747_b200 import make_mlp, qp
order = int(os.environ.get("ORDER", 1))
reps = int(os.environ.get("REPS", 200))
m = make_mlp([17] + [512] * 12 + [6], "silu", "full", 12512)
b = qp.QpBuilder(m, latency_mode=1)
cfg = qp.OcpConfig(horizon=20, dt=0.02, q_diag=np.ones(13), r_diag=np.full(4, .1), taylor_order=order)
x, u, rx, ru = bench._quad_iterate(np, 1, 20, 3)
p = qp.QuadParams()
ts = []
for i in range(reps):
    t0 = time.perf_counter()
    b.cycle_qp(p, cfg, x, u, rx, ru)
    ts.append((time.perf_counter() - t0) * 1e6)
ts = sorted(ts[10:])
print("order", order, "p50 us", ts[len(ts) // 2])
