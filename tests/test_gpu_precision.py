"""Precision modes on WELL-CONDITIONED nets (hidden weights scaled so f and J
are O(1); 1/√fan_in-initialised deep nets are nearly constant and would hide
operand-rounding error). Metric: ‖a−b‖∞/(1+‖b‖∞) per node and block, max
over nodes (proj/tests/oracles.hpp:30-32) vs the fp64 oracle.

North-star bounds: 1e-5 in 3xTF32 (fp32-grade), 1e-3 in TF32 / bf16. Measured
on B200 (scripts/precision_probe.py), max over f, A, B:
                 12x512 g2.5  12x512 g2.0  5x256 g2.5  5x256 g2.0  5x256 g1.5  2x64 tanh g3
  3xtf32 :       7.2e-6       2.1e-7       2.2e-6      1.2e-6      2.6e-7      2.9e-7
  bf16x3 :       6.0e-5       1.4e-6       3.5e-5      1.2e-5      —           8.3e-6
  tf32   :       2.7e-3       4.4e-5       2.4e-3      1.3e-3      1.1e-4      6.3e-4
3xTF32 and bf16x3 meet their bounds on every net; single-pass TF32 meets 1e-3
except on the nets with |J| ~ 1 and depth (12x512 g2.5, 5x256 g >= 2), where
tf32 operand rounding (2^-11) accumulates to ~2.5e-3 — asserted below as a
documented limit (< 5e-3), not as a pass of the 1e-3 bound. The bench line
reports the per-mode figures on its own inputs and on these nets.
"""
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


def _err(om, prec, k, kernel, monkeypatch, seed=2203):
    monkeypatch.setenv("RTN_KERNEL", kernel)
    z = oracle.quad_nodes(seed, k)
    f, j, _ = om.batched_eval(z, 1)
    got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, 1)
    assert np.isfinite(got.values).all() and np.isfinite(got.jacobians).all()
    return max(oracle.max_node_rel_error(got.values, f),
               oracle.max_node_rel_error(got.jacobians[:, :, :13], j[:, :, :13]),
               oracle.max_node_rel_error(got.jacobians[:, :, 13:], j[:, :, 13:]))


CASES = [
    ([17] + [256] * 5 + [6], "silu", 2.0),   # cfg2/cfg4 shape
    ([17] + [256] * 5 + [6], "silu", 2.5),
    ([17] + [512] * 12 + [6], "silu", 2.0),  # cfg3/cfg5 shape
    ([17] + [512] * 12 + [6], "silu", 2.5),  # |J| ~ 2: the conditioned deep net
    ([17, 64, 64, 6], "tanh", 3.0),          # cfg1 shape
]
BOUND = {"3xtf32": 1e-5, "bf16x3": 1e-4}


@pytest.mark.parametrize("kernel", ["pair", "latency", "quad"])
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("prec", ["3xtf32", "bf16x3"])
def test_split_modes_on_conditioned_nets(prec, case, kernel, monkeypatch):
    """quad: the 4-CTA latency kernel (rtn_quad.cuh) runs every mode at width 512;
    other shapes fall back to the pair latency kernel. pair: 512 nodes."""
    sizes, act, gain = CASES[case]
    err = _err(_net(sizes, act, gain), prec, 512 if kernel == "pair" else 20, kernel, monkeypatch)
    assert err < BOUND[prec], f"{prec} {kernel} {sizes[1]}x{len(sizes) - 2} gain {gain}: {err:.2e}"


@pytest.mark.parametrize("kernel", ["pair", "latency", "quad"])
def test_3xtf32_at_the_conditioned_cfg3_net_holds_1e5(kernel, monkeypatch):
    """The acceptance case of the fp32-grade mode: 12x512 SiLU at gain 2.5, f/A/B
    each < 1e-5 (was 1.2e-5 with two main accumulators; four now, rtn_pair.cuh)."""
    err = _err(_net([17] + [512] * 12 + [6], "silu", 2.5), "3xtf32", 64 if kernel == "pair" else 20, kernel,
               monkeypatch)
    assert err < 1e-5, err


@pytest.mark.parametrize("kernel", ["pair", "latency", "quad", "rows", "split"])
def test_tf32_north_star_bound_where_it_holds(kernel, monkeypatch):
    """Single-pass TF32 at 1e-3 on the nets where tf32 operand rounding stays
    below it (shallow, or |J| well below 1)."""
    k = 2048 if kernel in ("pair", "rows", "split") else 20
    assert _err(_net([17, 64, 64, 6], "tanh", 3.0), "tf32", k, kernel, monkeypatch) < 1e-3
    assert _err(_net([17] + [256] * 5 + [6], "silu", 1.5), "tf32", k, kernel, monkeypatch) < 1e-3
    if kernel != "rows":
        assert _err(_net([17] + [512] * 12 + [6], "silu", 2.0), "tf32", k, kernel, monkeypatch) < 1e-3


@pytest.mark.parametrize("kernel", ["pair", "quad", "rows", "split"])
def test_tf32_documented_limit_on_deep_conditioned_nets(kernel, monkeypatch):
    """At |J| ~ 1 and depth (12x512 g2.5, 5x256 g2.0-2.5) single-pass TF32 reaches
    ~2.5e-3: the recorded limitation of the mode (use 3xTF32 for fp32-grade
    results). Guards against regression, does not claim the 1e-3 bound."""
    k = 4096 if kernel in ("pair", "rows", "split") else 20
    if kernel != "rows":
        assert _err(_net([17] + [512] * 12 + [6], "silu", 2.5), "tf32", k, kernel, monkeypatch) < 5e-3
    if kernel not in ("quad", "split"):
        assert _err(_net([17] + [256] * 5 + [6], "silu", 2.0), "tf32", k, kernel, monkeypatch) < 3e-3
        assert _err(_net([17] + [256] * 5 + [6], "silu", 2.5), "tf32", k, kernel, monkeypatch) < 5e-3


def test_rows_kernel_conditioned_nets_every_activation(monkeypatch):
    """rtn_rows.cuh (the cfg4 TF32 kernel, ex2/rcp SiLU) on conditioned nets with
    K >= 10k (many tiles per CTA pair) for tanh and SiLU. (ReLU is left to the
    parity tests on small batches: at 12k nodes x 1,280 neurons some
    pre-activations sit within TF32 rounding of 0, where ReLU's slope jumps
    0 <-> 1 and J is discontinuous — measured 7.5e-3, the reference's own ReLU
    check only uses FD at 1e-4, proj/tests/test_neural.cpp:59-68.)"""
    for act, gain in (("silu", 1.5), ("tanh", 1.5)):
        err = _err(_net([17] + [256] * 5 + [6], act, gain), "tf32", 12000, "rows", monkeypatch, seed=31)
        assert err < 1e-3, (act, err)


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


@pytest.mark.parametrize("prec", ["tf32", "3xtf32"])
def test_inputs_far_from_zero(prec, monkeypatch):
    """in_mean and z shifted by +20 (|z| >> in_scale): the kernels subtract the
    mean in fp64 before layer 0 (rtn_kernel.cuh load_z), so the result matches
    the unshifted case's accuracy instead of cancelling in an fp32 bias."""
    errs = []
    for shift in (0.0, 20.0):
        om = _net([17, 64, 64, 6], "tanh", 3.0)
        if shift:
            im, isc, omn, osc = om.norm()
            om.set_norm(im + shift, isc, omn, osc)
        monkeypatch.setenv("RTN_KERNEL", "pair")
        z = oracle.quad_nodes(2203, 256) + shift
        f, j, _ = om.batched_eval(z, 1)
        got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, 1)
        errs.append(max(oracle.max_node_rel_error(got.values, f), oracle.max_node_rel_error(got.jacobians, j)))
    assert errs[1] < 2 * errs[0] + 1e-7, errs


@pytest.mark.parametrize("kernel", ["pair", "latency", "quad", "rowsb"])
def test_bf16_single_pass_documented_bounds(kernel, monkeypatch):
    """Single-pass BF16 (RTN_BF16: bf16 operands, one kind::f16 pass, 2x the tf32
    MMA rate): 8-bit mantissa operand rounding, ~8x the TF32 error. It meets the
    1e-3 bound where |J| is well below 1 (12x512 g2.0: 3.2e-4; 5x256 g1.5: 8.9e-4)
    and reaches ~3e-2 on the |J| ~ 2 net — measured limits asserted here."""
    k = 2048 if kernel in ("pair", "rowsb") else 20
    assert _err(_net([17] + [512] * 12 + [6], "silu", 2.0), "bf16", k, kernel, monkeypatch) < 1e-3
    assert _err(_net([17] + [512] * 12 + [6], "silu", 1.0), "bf16", k, kernel, monkeypatch) < 1e-6
    assert _err(_net([17] + [512] * 12 + [6], "silu", 2.5), "bf16", k, kernel, monkeypatch) < 5e-2
    if kernel != "quad":
        assert _err(_net([17] + [256] * 5 + [6], "silu", 1.5), "bf16", k, kernel, monkeypatch) < 1.5e-3
        assert _err(_net([17, 64, 64, 6], "tanh", 3.0), "bf16", k, kernel, monkeypatch) < 1e-2
