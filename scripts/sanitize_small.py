"""Small device workload for compute-sanitizer (one tool per run): every kernel
family once on tiny batches (pair, latency, quad, rows, order 2 generic and
quadrotor tiles, 3xTF32, blocks + feedback through the fused cycle)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2203_07747_b200 import _lib  # noqa: E402

for sizes, act, k, kern, order, prec in (([17, 64, 64, 6], "tanh", 10, "pair", 1, "tf32"),
                                          ([17] + [512] * 3 + [6], "silu", 6, "quad", 1, "tf32"),
                                          ([17] + [512] * 3 + [6], "silu", 6, "latency", 1, "3xtf32"),
                                          ([17] + [256] * 3 + [6], "silu", 300, "rows", 1, "tf32"),
                                          ([17] + [256] * 3 + [6], "silu", 600, "pair", 1, "bf16"),
                                          ([17] + [256] * 2 + [6], "silu", 3, "pair", 2, "tf32"),
                                          ([6, 32, 32, 4], "tanh", 3, "pair", 2, "3xtf32")):
    os.environ["RTN_KERNEL"] = kern
    om = oracle.OracleModel.random_net(sizes, act, 1, True)
    z = oracle.quad_nodes(3, k) if sizes[0] == 17 else np.random.default_rng(1).uniform(-1, 1, (k, sizes[0]))
    got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, order)
    f, j, _ = om.batched_eval(z, order)
    print(kern, prec, order, "err", oracle.max_node_rel_error(got.values, f), flush=True)
print("done")
