"""TF32 error of the device path vs the fp64 oracle on well-conditioned nets."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
from paper_2203_07747_b200 import mlp_batched_eval, EvalOrder

def net(sizes, act, gain, seed=11):
    om = oracle.OracleModel.random_net(sizes, act, seed, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    return om

for kern in ("single", "pair"):
    os.environ["RTN_KERNEL"] = kern
    for sizes, act, gains in (([17]+[512]*12+[6], "silu", (1.0, 2.0, 2.5, 3.0)), ([17]+[256]*5+[6], "silu", (1.0, 2.0, 2.5, 3.0)), ([17, 64, 64, 6], "tanh", (1.0, 2.0, 3.0))):
        for g in gains:
            om = net(sizes, act, g)
            z = oracle.quad_nodes(2203, 64)
            f, j, _ = om.batched_eval(z, 1)
            got = mlp_batched_eval(oracle.to_product_model(om), z, EvalOrder.JACOBIAN)
            print(f"{kern:6s} {sizes[1]}x{len(sizes)-2} {act} gain {g}: |J|max {abs(j).max():8.3g}  err f {oracle.max_node_rel_error(got.values, f):.2e}  A {oracle.max_node_rel_error(got.jacobians[:,:,:13], j[:,:,:13]):.2e}  B {oracle.max_node_rel_error(got.jacobians[:,:,13:], j[:,:,13:]):.2e}", flush=True)
