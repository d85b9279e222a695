"""Precision modes on WELL-CONDITIONED nets (hidden weights scaled so f and J
are O(1); 1/√fan_in-initialised deep nets are nearly constant and would hide
operand-rounding error). Metric: ‖a−b‖∞/(1+‖b‖∞) per node and block, max
over nodes (proj/tests/oracles.hpp:30-32) vs the fp64 oracle.

Measured on B200 (scripts/precision_probe.py):
  tf32   : 12x512 2.2e-3, 5x256 2.3e-3, 2x64 4e-4   (1e-3 bound NOT met on deep conditioned nets)
  bf16x3 : 12x512 6e-5,   5x256 2e-5,   2x64 5e-6   (1e-3 class, ~20x margin)
  3xtf32 : 12x512 7e-5,   5x256 1e-5,   2x64 1e-6   (1e-5 on the cfg4 shape)
"""
import os

import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import _lib

pytestmark = pytest.mark.gpu


def _net(sizes, act, gain, seed=11):
    om = oracle.OracleModel.random_net(sizes, act, seed, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    return om


def _err(om, prec, k, kernel, monkeypatch):
    monkeypatch.setenv("RTN_KERNEL", kernel)
    z = oracle.quad_nodes(2203, k)
    f, j, _ = om.batched_eval(z, 1)
    got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, 1)
    assert np.isfinite(got.values).all() and np.isfinite(got.jacobians).all()
    return max(oracle.max_node_rel_error(got.values, f),
               oracle.max_node_rel_error(got.jacobians[:, :, :13], j[:, :, :13]),
               oracle.max_node_rel_error(got.jacobians[:, :, 13:], j[:, :, 13:]))


CASES = [
    # (sizes, act, gain, {prec: bound})
    ([17] + [256] * 5 + [6], "silu", 2.0, {"3xtf32": 1e-5, "bf16x3": 1e-4}),   # cfg4 shape
    ([17] + [256] * 5 + [6], "silu", 2.5, {"3xtf32": 2e-5, "bf16x3": 1e-4}),
    ([17] + [512] * 12 + [6], "silu", 2.5, {"3xtf32": 2e-4, "bf16x3": 2e-4}),  # cfg3/cfg5 shape
    ([17, 64, 64, 6], "tanh", 3.0, {"3xtf32": 1e-5, "bf16x3": 2e-5}),          # cfg1 shape
]


@pytest.mark.parametrize("kernel", ["pair", "latency"])
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("prec", ["3xtf32", "bf16x3"])
def test_split_modes_on_conditioned_nets(prec, case, kernel, monkeypatch):
    sizes, act, gain, bounds = CASES[case]
    err = _err(_net(sizes, act, gain), prec, 64 if kernel == "pair" else 20, kernel, monkeypatch)
    assert err < bounds[prec], f"{prec} {sizes[1]}x{len(sizes) - 2}: {err:.2e}"


def test_tf32_documented_bound_on_conditioned_nets(monkeypatch):
    """Single-pass TF32 keeps < 1e-3 on shallow nets; deep conditioned nets
    reach ~2e-3 (recorded limitation) — guard against regression."""
    assert _err(_net([17, 64, 64, 6], "tanh", 3.0), "tf32", 64, "pair", monkeypatch) < 1e-3
    assert _err(_net([17] + [512] * 12 + [6], "silu", 2.5), "tf32", 64, "pair", monkeypatch) < 5e-3


@pytest.mark.parametrize("prec", ["3xtf32", "bf16x3"])
def test_split_modes_batch_invariance(prec, monkeypatch):
    """Within one kernel variant a node's result does not depend on the batch."""
    monkeypatch.setenv("RTN_KERNEL", "pair")
    om = _net([17] + [256] * 3 + [6], "silu", 2.0)
    eng = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec])
    z = oracle.quad_nodes(5, 29)
    full = eng.prepare(z, 1)
    for i in (0, 7, 28):
        one = eng.prepare(z[i:i + 1], 1)
        assert np.array_equal(one.values[0], full.values[i]) and np.array_equal(one.jacobians[0], full.jacobians[i])
