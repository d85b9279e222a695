"""Precision modes on WELL-CONDITIONED nets (hidden weights scaled so f and J
are O(1); 1/√fan_in-initialised deep nets are nearly constant and would hide
operand-rounding error). Metric: ‖a−b‖∞/(1+‖b‖∞) per node and block, max
over nodes (proj/tests/oracles.hpp:30-32) vs the fp64 oracle.

Measured on B200 (scripts/precision_probe.py), max over f, A, B:
                 12x512 g2.0  12x512 g2.5  5x256 g2.5  2x64 tanh g3
  tf32   :       3.4e-5       2.2e-3       2.3e-3      4.4e-4
  bf16x3 :       1.4e-6       6.0e-5       2.0e-5      5.0e-6
  3xtf32 :       2.8e-7       1.2e-5       2.1e-6      2.3e-7
Gain 2.5 at depth 12 is the edge of the net's stable regime: 1e-7 relative
noise on every activation moves f by 6e-7 there and by 8e-9 at gain 2.0 (numpy
fp64 check; plain numpy fp32 reaches 1.2e-6 at gain 2.5), so the north-star
bounds (1e-3 tf32/bf16, 1e-5 3xtf32) are asserted at gain 2.0 and the gain-2.5
figures are regression guards. 3xTF32 accumulates its correction passes and the
odd chunks of its main pass in separate TMEM accumulators (rtn_pair.cuh kCorr,
kSplitMain): 7e-5 -> 1.2e-5 at 12x512 g2.5.
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
    ([17] + [256] * 5 + [6], "silu", 2.5, {"3xtf32": 5e-6, "bf16x3": 1e-4}),
    ([17] + [512] * 12 + [6], "silu", 2.0, {"3xtf32": 1e-5, "bf16x3": 1e-5}),  # cfg3/cfg5 shape
    ([17] + [512] * 12 + [6], "silu", 2.5, {"3xtf32": 3e-5, "bf16x3": 2e-4}),  # edge of stability
    ([17, 64, 64, 6], "tanh", 3.0, {"3xtf32": 1e-6, "bf16x3": 2e-5}),          # cfg1 shape
]


@pytest.mark.parametrize("kernel", ["pair", "latency", "quad"])
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("prec", ["3xtf32", "bf16x3"])
def test_split_modes_on_conditioned_nets(prec, case, kernel, monkeypatch):
    """quad: the 4-CTA latency kernel (rtn_quad.cuh) also runs bf16x3 and 3xTF32 at
    width 512; other shapes fall back to the pair latency kernel."""
    sizes, act, gain, bounds = CASES[case]
    err = _err(_net(sizes, act, gain), prec, 64 if kernel == "pair" else 20, kernel, monkeypatch)
    assert err < bounds[prec], f"{prec} {sizes[1]}x{len(sizes) - 2}: {err:.2e}"


def test_tf32_documented_bound_on_conditioned_nets(monkeypatch):
    """Single-pass TF32 keeps < 1e-3 on shallow nets and on 12x512 at gain 2.0;
    at gain 2.5 (edge of stability) it reaches ~2e-3 (recorded limitation,
    DESIGN.md §4) — guard against regression."""
    assert _err(_net([17, 64, 64, 6], "tanh", 3.0), "tf32", 64, "pair", monkeypatch) < 1e-3
    assert _err(_net([17] + [512] * 12 + [6], "silu", 2.0), "tf32", 64, "pair", monkeypatch) < 1e-4
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
