"""Reverse-mode Jacobians (rtn_reverse.cuh) vs the oracle, and the cfg5-shape
device time of forward vs reverse mode. Usage: [DEPTH=12] [K=3000] python scripts/reverse_check.py"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from paper_2203_07747_b200 import _lib  # noqa: E402

k = int(os.environ.get("K", "3000"))
depth = int(os.environ.get("DEPTH", "12"))
om = oracle.OracleModel.random_net([17] + [512] * depth + [6], os.environ.get("ACT", "silu"), 11, True)
for l, (w, b) in enumerate(om.layers()):
    if l < len(om.layers()) - 1:
        om.set_layer(l, w * float(os.environ.get("GAIN", "2.0")), b)
z = oracle.quad_nodes(3, k)
pm = oracle.to_product_model(om)
fwd = pm.engine().prepare(z, 1)
rev = pm.engine(jacobian_mode=1).prepare(z, 1)
idx = np.arange(0, k, 7)
f, j, _ = om.batched_eval(z[idx], 1)
for name, got in (("forward", fwd), ("reverse", rev)):
    print(name, "max err f", oracle.max_node_rel_error(got.values[idx], f), "J",
          oracle.max_node_rel_error(got.jacobians[idx], j), "finite", np.isfinite(got.values).all() and np.isfinite(got.jacobians).all(), flush=True)
