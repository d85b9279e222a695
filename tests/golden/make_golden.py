"""Generates tests/golden/*.json from the CPU oracle (oracle/), which restates
/root/reference/proj/src/neural.cpp and is pinned by the reference's own
known-answer tests (oracle/test_oracle.cpp). Fixtures are small, seeded and
committed so GPU tests can check against fixed numbers without rebuilding the
oracle's state; re-run this script to regenerate:

    python tests/golden/make_golden.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def dump(name, sizes, act, rng_seed, gain, k, z_seed, order):
    om = oracle.OracleModel.random_net(sizes, act, rng_seed, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    z = oracle.quad_nodes(z_seed, k) if sizes[0] == 17 else oracle_vector(z_seed, k, sizes[0])
    f, j, h = om.batched_eval(z, order)
    path = os.path.join(OUT, name + ".rmlp")
    om.save(path)
    os.remove(path + ".json")
    rec = {"model_file": name + ".rmlp", "sizes": sizes, "activation": act, "rng_seed": rng_seed, "gain": gain,
           "order": order, "z": z.tolist(), "f": f.tolist(), "jac": j.tolist()}
    if order == 2:
        rec["hess"] = h.tolist()
    with open(os.path.join(OUT, name + ".json"), "w") as fh:
        json.dump(rec, fh)


def oracle_vector(seed, k, n):
    import numpy as np
    return np.random.default_rng(seed).uniform(-2, 2, (k, n))


if __name__ == "__main__":
    # cfg1: the one configuration the reference's own arithmetic (tanh) covers
    dump("cfg1_tanh_2x64_N10", [17, 64, 64, 6], "tanh", 11, 2.0, 10, 2203, 1)
    # a conditioned SiLU net (gain keeps f and J at O(1)) and a second-order case
    dump("silu_3x128_N8", [17, 128, 128, 128, 6], "silu", 12, 2.5, 8, 2204, 2)
    # the reference's test shape {6,32,32,4} (proj/tests/test_neural.cpp:119-145)
    dump("tanh_6_32_32_4_K13", [6, 32, 32, 4], "tanh", 23, 1.0, 13, 23, 2)
    print("ok")
