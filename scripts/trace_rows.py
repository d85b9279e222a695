"""Event timeline of pair 0's first two tiles in the rows kernel (RTN_TRACE)."""
import ctypes as C, os, sys
os.environ["RTN_TRACE"] = "1"
os.environ["RTN_KERNEL"] = "rows"
sys.path.insert(0, ".")
import numpy as np
from paper_2203_07747_b200 import _lib, make_mlp, synth_quad_nodes, mlp_batched_eval, EvalOrder
sizes = [17] + [256] * 5 + [6]
k = int(sys.argv[1]) if len(sys.argv) > 1 else 81920
m = make_mlp(sizes, "silu", "full", 5256)
z = synth_quad_nodes(7, k)
for _ in range(3):
    mlp_batched_eval(m, z, EvalOrder.JACOBIAN)
L = _lib.lib()
buf = (C.c_ulonglong * 256)()
L.rtn_debug_trace(buf, 256)
t = np.array(buf, dtype=np.float64)
t0 = t[64]
rel = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")
n_mma = len(sizes) - 3
for tix in range(2):
    for li in range(n_mma + 1):
        b = tix * 24 + li * 3
        print(f"tile {tix} MMA layer {li}: start {rel(t[b]):8.3f} act0 {rel(t[b+1]):8.3f} issued {rel(t[b+2]):8.3f} us")
    for L in range(n_mma + 1):
        row = []
        for r in range(2):
            for h in range(2):
                i = 64 + (((r * 2 + h) * 2 + tix) * 6 + L) * 3
                row.append(f"c{r}h{h} {rel(t[i]):7.3f}/{rel(t[i+1]):7.3f}/{rel(t[i+2]):7.3f}")
        print(f"tile {tix} epi L{L}: " + " | ".join(row))
for h in range(2):
    c = t[216 + h * 12: 216 + h * 12 + 4]
    print(f"fine h{h} (cycles from tmem_full seen): " + " ".join(f"{x - c[0]:.0f}" for x in c))
print("  points: 0 full seen, 1 table stage 0, 2 chunk 0 published, 3 all published")
