"""Second order on the device (cfg3: 12x512 SiLU, N=20, first AND second
order): f, J and the per-output Hessians vs the oracle's HessianSingle
(proj/src/neural.cpp:175-225, generalised to SiLU). Tolerance metric as in
proj/tests/oracles.hpp:30-32, per node and block, max over nodes."""
import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import (UnsupportedError, _lib, eval_taylor, eval_taylor_jacobian, make_mlp,
                                   mlp_batched_eval, EvalOrder, prepare_nodes)

pytestmark = pytest.mark.gpu


def _net(sizes, act, gain, seed=11):
    om = oracle.OracleModel.random_net(sizes, act, seed, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    return om


def _errs(om, prec, k=20):
    z = oracle.quad_nodes(2203, k)
    f, j, h = om.batched_eval(z, 2)
    got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, 2)
    assert np.isfinite(got.hessians).all()
    return (oracle.max_node_rel_error(got.values, f), oracle.max_node_rel_error(got.jacobians, j),
            oracle.max_node_rel_error(got.hessians, h), got)


# (sizes, act, gain, {prec: bound})  — bounds from scripts/precision_probe.py-style runs
CASES = [
    ([17] + [512] * 12 + [6], "silu", 2.5, {"tf32": 5e-3, "bf16x3": 3e-4, "3xtf32": 3e-4}),  # cfg3
    ([17] + [256] * 5 + [6], "silu", 2.5, {"tf32": 5e-3, "bf16x3": 1e-4, "3xtf32": 5e-5}),
    ([17, 64, 64, 6], "tanh", 2.0, {"tf32": 1e-3, "bf16x3": 2e-5, "3xtf32": 1e-5}),          # cfg1
    ([17] + [512] * 12 + [6], "silu", 1.0, {"tf32": 1e-3, "bf16x3": 1e-5, "3xtf32": 1e-5}),  # MakeMlp-scale
]


@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("prec", ["tf32", "bf16x3", "3xtf32"])
def test_order2_matches_oracle(prec, case):
    sizes, act, gain, bounds = CASES[case]
    ef, ej, eh, got = _errs(_net(sizes, act, gain), prec)
    assert max(ef, ej, eh) < bounds[prec], (prec, sizes[1], len(sizes) - 2, ef, ej, eh)
    # Hessians are exactly symmetric (one value written to (a,b) and (b,a))
    assert np.array_equal(got.hessians, np.swapaxes(got.hessians, 2, 3))


def test_order2_ragged_and_large_batch():
    om = _net([17] + [256] * 3 + [6], "silu", 2.0)
    for k in (1, 3, 151):
        ef, ej, eh, _ = _errs(om, "bf16x3", k)
        assert max(ef, ej, eh) < 1e-4


def test_order2_prepare_nodes_taylor_consistency():
    """PrepareNodes(order=2) on the device, then the host consumers
    (proj/src/taylor.cpp:57-74): expansion point exact, and the second-order
    expansion beats the first-order one at small steps (test_taylor.cpp:102-135)."""
    om = _net([17, 128, 128, 6], "silu", 2.0)
    m = oracle.to_product_model(om)
    eng_kw = dict(precision=_lib.RTN_3XTF32)
    z0 = oracle.quad_nodes(9, 4)
    a2 = prepare_nodes(m, z0, 2, **eng_kw)
    a1 = prepare_nodes(m, z0, 1, **eng_kw)
    rng = np.random.default_rng(0)
    for k in range(4):
        assert np.array_equal(eval_taylor(a2[k], z0[k]), a2[k].f_bar)
        assert np.array_equal(eval_taylor_jacobian(a2[k], z0[k]), a2[k].jac)
        d = rng.uniform(-1, 1, 17)
        d /= np.linalg.norm(d)
        z = z0[k] + 0.02 * d
        f_true, _, _ = om.batched_eval(z[None], 0)
        r1 = np.max(np.abs(eval_taylor(a1[k], z) - f_true[0]))
        r2 = np.max(np.abs(eval_taylor(a2[k], z) - f_true[0]))
        assert r2 < r1


def test_order2_unsupported_shapes():
    m = make_mlp([6, 32, 32, 4], "tanh", "full", 3)   # the device order-2 path is built for 17 inputs
    with pytest.raises(UnsupportedError):
        mlp_batched_eval(m, np.zeros((2, 6)), EvalOrder.HESSIAN)
