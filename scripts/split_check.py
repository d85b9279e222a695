"""Split kernel (rtn_split.cuh) vs the oracle on a conditioned 12x512 net, then
cfg5-shape device time of split vs pair (RTN_KERNEL). Usage: python scripts/split_check.py [K]"""
import ctypes as C
import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2203_07747_b200 import _lib  # noqa: E402

os.environ["RTN_KERNEL"] = os.environ.get("RTN_KERNEL", "split")
k = int(os.environ.get("K", "3000"))
if os.environ.get("RTN_TRACE_HOST"):
    import threading, time
    os.environ["RTN_TRACE"] = "1"

    def _watch():
        time.sleep(float(os.environ.get("WATCH_S", "15")))
        buf = (C.c_ulonglong * 64)()
        _lib.lib().rtn_debug_trace(buf, 64)
        print("producer", [hex(buf[i]) for i in range(2)], "mma wait-act", hex(buf[2]), "mma wait-full", hex(buf[3]))
        print("epilogue CTA0", list(buf[8:16]), "CTA1", list(buf[16:24]), flush=True)
        os._exit(3)
    threading.Thread(target=_watch, daemon=True).start()
om = oracle.OracleModel.random_net([17] + [512] * int(os.environ.get("DEPTH", "12")) + [6], "silu", 11, True)
for l, (w, b) in enumerate(om.layers()):
    if l < len(om.layers()) - 1:
        om.set_layer(l, w * float(os.environ.get("GAIN", "2.0")), b)
z = oracle.quad_nodes(3, k)
got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS.get(os.environ.get("PREC", "tf32"), None) or int(os.environ.get("PREC", "0"))).prepare(z, 1)
idx = np.arange(0, k, 7)
f, j, _ = om.batched_eval(z[idx], 1)
print(os.environ["RTN_KERNEL"], "max err f", oracle.max_node_rel_error(got.values[idx], f), "J",
      oracle.max_node_rel_error(got.jacobians[idx], j), "finite", np.isfinite(got.values).all(), flush=True)
