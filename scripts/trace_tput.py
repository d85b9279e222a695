"""Event timeline of one tile of CTA pair 0 in the throughput kernel (RTN_TRACE
= 1 + tile index): per (layer, block) the MMA warp's issue window and each
CTA's epilogue (accumulator seen, input group free, published).
Usage: RTN_TRACE=3 [RTN_DEBUG=n] [ORDER=2] python scripts/trace_tput.py [K]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2203_07747_b200 import EvalOrder, _lib, make_mlp, mlp_batched_eval, synth_quad_nodes  # noqa: E402

os.environ.setdefault("RTN_TRACE", "3")
sizes = [17] + [512] * 12 + [6]
k = int(sys.argv[1]) if len(sys.argv) > 1 else 409600
m = make_mlp(sizes, "silu", "full", 12512)
z = synth_quad_nodes(7, k)
order = EvalOrder.HESSIAN if os.environ.get("ORDER") == "2" else EvalOrder.JACOBIAN
for _ in range(3):
    mlp_batched_eval(m, z, order)
buf = (C.c_ulonglong * 256)()
_lib.lib().rtn_debug_trace(buf, 256)
t = np.array(buf, dtype=np.float64)
t0 = t[0]
rel = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")
print(f"RTN_TRACE={os.environ['RTN_TRACE']} RTN_DEBUG={os.environ.get('RTN_DEBUG', '0')} K={k} (us from layer-1 block-0 issue)")
for r in range(2):
    b = [rel(t[180 + r * 6 + e]) for e in range(4)]
    print(f"tile start CTA{r}: top {b[0]:8.2f} layer0 math done {b[1]:8.2f} prev output done {b[2]:8.2f} "
          f"outputs written {b[3]:8.2f} layer0 published {rel(t[192 + r]):8.2f}")
prev_end = None
for l in range(11):
    for mb in range(2):
        i = l * 2 + mb
        e0 = [rel(t[48 + i * 3 + q]) for q in range(3)]
        e1 = [rel(t[114 + i * 3 + q]) for q in range(3)]
        print(f"L{l + 1} mb{mb}: mma issue {rel(t[i * 2]):8.2f}-{rel(t[i * 2 + 1]):8.2f} | CTA0 acc {e0[0]:8.2f} "
              f"free {e0[1]:8.2f} pub {e0[2]:8.2f} | CTA1 acc {e1[0]:8.2f} free {e1[1]:8.2f} pub {e1[2]:8.2f}")
print(f"output MMAs issued {rel(t[44]):8.2f}; hidden layers done CTA0 {rel(t[194]):8.2f} CTA1 {rel(t[195]):8.2f}")
