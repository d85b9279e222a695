"""Quad latency kernel smoke: RTN_KERNEL=quad vs oracle and vs the pair latency kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_2203_07747_b200 import _lib
om = oracle.OracleModel.random_net([17] + [512] * int(os.environ.get("L", 12)) + [6], "silu", 3, True)
for k in [int(x) for x in os.environ.get("KS", "1,2,20").split(",")]:
    z = oracle.quad_nodes(5, k)
    f, j, _ = om.batched_eval(z, 1)
    res = {}
    for kern in ("quad", "latency"):
        os.environ["RTN_KERNEL"] = kern
        m = oracle.to_product_model(om)
        got = m.engine().prepare(z, 1)
        res[kern] = got
        print(kern, k, "err f %.2e J %.2e" % (oracle.max_node_rel_error(got.values, f), oracle.max_node_rel_error(got.jacobians, j)), flush=True)
    print("quad vs latency max diff", np.abs(res["quad"].jacobians - res["latency"].jacobians).max(), flush=True)
