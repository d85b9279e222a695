"""MMA-issue timeline of one tile of CTA pair 0 in the split kernel (rtn_split.cuh):
per hidden layer the issue start of blocks B0..B3 and the end of B3's issue.
Usage: RTN_TRACE=3 [RTN_DEBUG=128] python scripts/trace_split.py [K]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2203_07747_b200 import EvalOrder, _lib, make_mlp, mlp_batched_eval, synth_quad_nodes  # noqa: E402

os.environ.setdefault("RTN_TRACE", "3")
os.environ.setdefault("RTN_KERNEL", "split")
k = int(sys.argv[1]) if len(sys.argv) > 1 else 409600
m = make_mlp([17] + [512] * 12 + [6], "silu", "full", 12512)
z = synth_quad_nodes(7, k)
for _ in range(3):
    mlp_batched_eval(m, z, EvalOrder.JACOBIAN)
buf = (C.c_ulonglong * 256)()
_lib.lib().rtn_debug_trace(buf, 256)
t = np.array(buf[:55], dtype=np.float64).reshape(11, 5)
t0 = t[0, 0]
print(f"RTN_DEBUG={os.environ.get('RTN_DEBUG', '0')} K={k}: us from layer-1 B0 issue; columns B0 B1 B2 B3 B3-end, then per-block durations")
for l in range(11):
    r = (t[l] - t0) / 1e3
    d = np.diff(t[l]) / 1e3
    nxt = ((t[l + 1, 0] - t[l, 4]) / 1e3) if l < 10 else float("nan")
    print(f"L{l + 1:2d}: " + " ".join(f"{x:8.2f}" for x in r) + " | " + " ".join(f"{x:5.2f}" for x in d) +
          f" | gap to next layer {nxt:5.2f}")
if not int(os.environ.get("RTN_DEBUG", "0")) & 128:
    e = np.array(buf[64:174], dtype=np.float64).reshape(11, 10)
    print("epilogue CTA0 (us from layer-1 B0 issue): B0 seen/done, B1 seen/done, B2 seen/done, s_free seen, S stored, B3 seen/done")
    for l in range(11):
        print(f"L{l + 1:2d}: " + " ".join(f"{(x - t0) / 1e3:8.2f}" for x in e[l]))
    tbv = np.array(buf[180:192], dtype=np.float64)
    base = t[10, 4]
    print("tile boundary (us from L11 B3 issue end): out seen", f"{(tbv[0] - base) / 1e3:.2f}", "out written",
          f"{(tbv[1] - base) / 1e3:.2f}", "layer0 start", f"{(tbv[2] - base) / 1e3:.2f}",
          "quarters (tables, stored):", " ".join(f"{(x - base) / 1e3:.2f}" for x in tbv[3:11]))
    ch = np.array(buf[200:232], dtype=np.float64).reshape(16, 2)
    b0 = t[4, 0]
    print("L5 B0 per chunk (us from its issue start): act-ready / weights-ready")
    print(" ".join(f"{(a - b0) / 1e3:.2f}/{(b - b0) / 1e3:.2f}" for a, b in ch))
