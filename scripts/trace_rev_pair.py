"""MMA-issue and epilogue timeline (RTN_TRACE) of one tile of CTA pair 0 in the
pair kernel's reverse value / adjoint passes.
Usage: RTN_TRACE=3 RTN_TRACE_PASS=0|1 PREC=3xtf32 python scripts/trace_rev_pair.py [K]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2203_07747_b200 import _lib, make_mlp, synth_quad_nodes  # noqa: E402

os.environ.setdefault("RTN_TRACE", "3")
k = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
w, d = int(os.environ.get("WIDTH", "512")), int(os.environ.get("DEPTH", "12"))
m = make_mlp([17] + [w] * d + [6], "silu", "full", 12512)
eng = m.engine(precision=_lib.PRECISIONS[os.environ.get("PREC", "3xtf32")], jacobian_mode=1)
z = synth_quad_nodes(7, k)
for _ in range(2):
    eng.prepare(z, 1)
buf = (C.c_ulonglong * 256)()
_lib.lib().rtn_debug_trace(buf, 256)
t = np.array(buf[:], dtype=np.float64)
t0 = t[0]
us = lambda x: (x - t0) / 1e3 if x else float("nan")  # noqa: E731
pas = os.environ.get("RTN_TRACE_PASS", "1")
print(f"pass {pas} ({'value' if pas == '0' else 'adjoint'}); times in us from the first MMA issue")
for r in range(2):
    print(f"rank {r}: first_store {us(t[192 + r]):8.2f} .. {us(t[194 + r]):8.2f}")
print("layer/block: MMA issue start, end | rank0 epi: acc ready, act done, published | rank1 ...")
for i in range(min(22, 2 * (d - 1))):
    e = [us(t[48 + r * 66 + i * 3 + c]) for r in range(2) for c in range(3)]
    print(f"L{i // 2 + 1} mb{i % 2}: {us(t[2 * i]):8.2f} {us(t[2 * i + 1]):8.2f} |"
          + " ".join(f"{x:8.2f}" for x in e[:3]) + " |" + " ".join(f"{x:8.2f}" for x in e[3:]))
