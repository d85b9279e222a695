import sys; sys.path.insert(0, ".")
import numpy as np, oracle
from oracle import OracleModel, max_node_rel_error, to_product_model
for sizes, act in (([24, 400, 512, 16], "relu"), ([24, 400, 512, 16], "silu"), ([17, 512, 512, 6], "relu"), ([24, 512, 512, 6], "silu"), ([17, 400, 512, 16], "silu")):
    om = OracleModel.random_net(sizes, act, 11, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2: om.set_layer(l, w * 1.5, b)
    z = np.random.default_rng(2203).uniform(-2, 2, (2000, sizes[0])) if sizes[0] != 17 else oracle.quad_nodes(2203, 2000)
    f, j, _ = om.batched_eval(z, 1)
    pm = to_product_model(om)
    for jm in (0, 1):
        g = pm.engine(jacobian_mode=jm).prepare(z, 1)
        e = np.array([max_node_rel_error(g.jacobians[i:i+1], j[i:i+1]) for i in range(len(z))])
        print(sizes, act, "mode", jm, "J err max", e.max(), "nodes > 1e-3:", int((e > 1e-3).sum()))
