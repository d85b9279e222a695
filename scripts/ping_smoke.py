"""Width-256 ping-pong kernel smoke: vs oracle and vs the pair kernel (RTN_PINGPONG=0)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
L = int(os.environ.get("L", 5))
om = oracle.OracleModel.random_net([17] + [256] * L + [6], "silu", 3, True)
for k in [int(x) for x in os.environ.get("KS", "1184,2000,4736").split(",")]:
    z = oracle.quad_nodes(5, k)
    f, j, _ = om.batched_eval(z, 1)
    res = {}
    for pp in ("1", "0"):
        os.environ["RTN_PINGPONG"] = pp
        m = oracle.to_product_model(om)
        got = m.engine().prepare(z, 1)
        res[pp] = got
        print("pingpong" if pp == "1" else "pair    ", k, "err f %.2e J %.2e" % (oracle.max_node_rel_error(got.values, f), oracle.max_node_rel_error(got.jacobians, j)), flush=True)
    print("  max diff", np.abs(res["1"].jacobians - res["0"].jacobians).max(), flush=True)
