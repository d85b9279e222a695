"""rtn_rowsa.cuh quick check: parity vs the fp64 oracle and device time at the cfg5 shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402

os.environ["RTN_KERNEL"] = "rowsa"
for sizes, act, gain, k in (([17, 512, 512, 6], "silu", 2.0, 7), ([17] + [512] * 12 + [6], "silu", 2.0, 20),
                             ([17] + [512] * 12 + [6], "silu", 2.0, 5000), ([7, 512, 512, 512, 3], "tanh", 1.5, 999),
                             ([17, 300, 400, 6], "silu", 1.5, 333)):
    om = oracle.OracleModel.random_net(sizes, act, 11, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    z = oracle.quad_nodes(2203, k) if sizes[0] == 17 else np.random.default_rng(2).uniform(-1, 1, (k, sizes[0]))
    f, j, _ = om.batched_eval(z, 1)
    got = oracle.to_product_model(om).engine().prepare(z, 1)
    print(sizes[:3], k, "err f %.2e J %.2e" % (oracle.max_node_rel_error(got.values, f),
                                              oracle.max_node_rel_error(got.jacobians, j)),
          "finite", bool(np.isfinite(got.jacobians).all()), flush=True)
