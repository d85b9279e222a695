"""Device error vs the fp64 oracle per precision mode and kernel, on
well-conditioned nets (hidden weights x gain so f and J are O(1)).

    python scripts/precision_probe.py            # ORDER=1|2, PRECS=tf32,3xtf32,bf16x3, KERNS=...

Prints one line per (mode, kernel, net): the max over nodes of the reference
metric ‖a−b‖∞/(1+‖b‖∞) (proj/tests/oracles.hpp:30-32) for f, A, B (and H).
MEAN_SHIFT=s adds s to in_mean and to the node rows (inputs far from 0
relative to in_scale: the layer-0 cancellation case)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from paper_2203_07747_b200 import _lib  # noqa: E402


def net(sizes, act, gain, seed=11, shift=0.0):
    om = oracle.OracleModel.random_net(sizes, act, seed, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    if shift:
        im, isc, omn, osc = om.norm()
        om.set_norm(im + shift, isc, omn, osc)
    return om


CASES = [([17] + [512] * 12 + [6], "silu", 2.5), ([17] + [512] * 12 + [6], "silu", 2.0),
         ([17] + [256] * 5 + [6], "silu", 2.5), ([17] + [256] * 5 + [6], "silu", 2.0),
         ([17, 64, 64, 6], "tanh", 3.0), ([17] + [512] * 12 + [6], "silu", 1.0), ([17] + [256] * 5 + [6], "silu", 1.5)]
K_OF = {"pair": 512, "latency": 20, "quad": 20, "rows": 2048}


GENERIC2 = [([6, 32, 32, 4], "tanh", 1.0), ([3, 16, 16, 2], "tanh", 1.0), ([7] + [256] * 3 + [3], "silu", 2.0),
            ([26, 256, 256, 3], "silu", 2.0), ([31, 128, 128, 5], "tanh", 1.5), ([3] + [512] * 12 + [3], "silu", 2.5),
            ([17] + [512] * 12 + [6], "silu", 2.5)]


def generic_order2():
    """Order 2 on the reference's own test shapes and the residual variants' widths."""
    for prec in os.environ.get("PRECS", "tf32,3xtf32,bf16x3").split(","):
        for sizes, act, g in GENERIC2:
            om = net(sizes, act, g)
            z = np.random.default_rng(5).uniform(-1, 1, (20, sizes[0]))
            f, j, h = om.batched_eval(z, 2)
            got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, 2)
            e = [oracle.max_node_rel_error(a, b) for a, b in ((got.values, f), (got.jacobians, j), (got.hessians, h))]
            sym = bool(np.array_equal(got.hessians, np.swapaxes(got.hessians, 2, 3)))
            print(f"{prec:6s} order2 {sizes}: f {e[0]:.2e} J {e[1]:.2e} H {e[2]:.2e} sym {sym} max {max(e):.2e}",
                  flush=True)


def main():
    if os.environ.get("GENERIC2"):
        return generic_order2()
    order = int(os.environ.get("ORDER", "1"))
    shift = float(os.environ.get("MEAN_SHIFT", "0"))
    for prec in os.environ.get("PRECS", "tf32,3xtf32,bf16x3").split(","):
        for kern in os.environ.get("KERNS", "pair,latency,quad,rows").split(","):
            os.environ["RTN_KERNEL"] = kern
            for sizes, act, g in CASES:
                if kern == "rows" and (sizes[1] != 256 or prec != "tf32"):
                    continue
                if kern == "quad" and sizes[1] != 512:
                    continue
                om = net(sizes, act, g, shift=shift)
                z = oracle.quad_nodes(2203, K_OF[kern]) + shift
                f, j, hh = om.batched_eval(z, order)
                got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, order)
                ef = oracle.max_node_rel_error(got.values, f)
                ea = oracle.max_node_rel_error(got.jacobians[:, :, :13], j[:, :, :13])
                eb = oracle.max_node_rel_error(got.jacobians[:, :, 13:], j[:, :, 13:])
                eh = oracle.max_node_rel_error(got.hessians, hh) if order == 2 else float("nan")
                jn = float(np.abs(j).max())
                print(f"{prec:6s} {kern:7s} {sizes[1]}x{len(sizes) - 2} {act} gain {g}: f {ef:.2e} A {ea:.2e} "
                      f"B {eb:.2e} H {eh:.2e} |J|max {jn:.2e} max {max(ef, ea, eb, 0 if order == 1 else eh):.2e}",
                      flush=True)


if __name__ == "__main__":
    main()
