"""Device error vs the fp64 oracle per precision mode and kernel, on
well-conditioned nets (hidden weights x gain so f and J are O(1))."""
import os, sys
sys.path.insert(0, ".")
import numpy as np
import oracle
from paper_2203_07747_b200 import _lib

def net(sizes, act, gain, seed=11):
    om = oracle.OracleModel.random_net(sizes, act, seed, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    return om

cases = [([17]+[512]*12+[6], "silu", 2.5), ([17]+[512]*12+[6], "silu", 2.0), ([17]+[256]*5+[6], "silu", 2.5), ([17, 64, 64, 6], "tanh", 3.0),
         ([17]+[512]*12+[6], "silu", 1.0)]
order = int(os.environ.get("ORDER", "1"))
for prec in os.environ.get("PRECS", "tf32,3xtf32,bf16x3").split(","):
    for kern in ("pair", "latency"):
        os.environ["RTN_KERNEL"] = kern
        for sizes, act, g in cases:
            om = net(sizes, act, g)
            z = oracle.quad_nodes(2203, 64 if kern == "pair" else 20)
            f, j, hh = om.batched_eval(z, order)
            m = oracle.to_product_model(om)
            got = m.engine(precision=_lib.PRECISIONS[prec]).prepare(z, order)
            ef = oracle.max_node_rel_error(got.values, f)
            ea = oracle.max_node_rel_error(got.jacobians[:, :, :13], j[:, :, :13])
            eb = oracle.max_node_rel_error(got.jacobians[:, :, 13:], j[:, :, 13:])
            eh = oracle.max_node_rel_error(got.hessians, hh) if order == 2 else float("nan")
            print(f"{prec:6s} {kern:7s} {sizes[1]}x{len(sizes)-2} {act} gain {g}: f {ef:.2e} A {ea:.2e} B {eb:.2e} H {eh:.2e}", flush=True)
