"""Reverse-mode Jacobians (rtn_ctx_set_jacobian_mode(ctx, 1); csrc/rtn_reverse.cuh):
the reference's own algorithm (BatchedCore's stacked reverse sweep,
proj/src/neural.cpp:132-163) on the tensor cores — a value pass that keeps each
layer's slope in an HBM scratch, then one adjoint row per output. Checked
against the fp64 oracle in the reference metric (proj/tests/oracles.hpp:30-32)
with the TF32 tolerances of the forward-mode tests, and against forward mode."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle
from oracle import OracleModel, max_node_rel_error, quad_nodes, to_product_model
from paper_2203_07747_b200 import _lib
from paper_2203_07747_b200.errors import raise_for_status

pytestmark = pytest.mark.gpu


def _net(sizes, act, gain, seed=11):
    om = OracleModel.random_net(sizes, act, seed, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    return om


def _z(n_in, k, seed=2203):
    return quad_nodes(seed, k) if n_in == 17 else np.random.default_rng(seed).uniform(-2, 2, (k, n_in))


def _errs(om, k, seed=2203):
    z = _z(om.sizes[0], k, seed)
    got = to_product_model(om).engine(jacobian_mode=1).prepare(z, 1)
    assert np.isfinite(got.values).all() and np.isfinite(got.jacobians).all()
    f, j, _ = om.batched_eval(z, 1)
    return max_node_rel_error(got.values, f), max_node_rel_error(got.jacobians, j), got


@pytest.mark.parametrize("k", [1, 255, 256, 257, 3001])
def test_reverse_mode_cfg3_shape_ragged(k):
    ef, ej, _ = _errs(_net([17] + [512] * 12 + [6], "silu", 2.0), k)
    assert ef < 1e-3 and ej < 1e-3, (ef, ej)


@pytest.mark.parametrize("sizes,act", [([17, 512, 6], "silu"), ([17, 512, 512, 6], "tanh"),
                                        ([7, 512, 512, 512, 3], "silu"), ([24, 400, 512, 16], "relu"),
                                        ([17] + [512] * 5 + [1], "silu"), ([3, 512, 512, 2], "tanh")])
def test_reverse_mode_shapes(sizes, act):
    """Input widths 3..24, outputs 1..16 (adjoint rows per CTA = 128 // n_out), 0-4
    hidden->hidden layers, hidden widths that pad to 512, every activation. ReLU's
    J jumps where a pre-activation is within TF32 rounding of 0 (forward mode
    shows the same nodes: ~100 of 2,000 here), so it is checked against forward
    mode, which takes the same slope decisions from the same value path."""
    om = _net(sizes, act, 1.5)
    if act == "relu":
        z = _z(sizes[0], 2000)
        pm = to_product_model(om)
        rev = pm.engine(jacobian_mode=1).prepare(z, 1)
        fwd = pm.engine().prepare(z, 1)
        assert np.array_equal(rev.values, fwd.values)
        assert max_node_rel_error(rev.jacobians, fwd.jacobians) < 1e-3
        return
    ef, ej, _ = _errs(om, 2000)
    assert ef < 1e-3 and ej < 1e-3, (sizes, act, ef, ej)


def test_reverse_mode_chunked_and_documented_limit():
    """More nodes than one scratch chunk (forced to 65,536 by RTN_REV_CHUNK; the
    default is a 2 GiB scratch in equal chunks): every chunk's J; and the |J| ~ 2
    edge-of-stability net, where TF32 (either algorithm) reaches ~3e-3."""
    om = _net([17] + [512] * 4 + [6], "silu", 1.5)
    z = quad_nodes(5, 70000)
    os.environ["RTN_REV_CHUNK"] = "65536"
    try:
        got = to_product_model(om).engine(jacobian_mode=1).prepare(z, 1)
    finally:
        del os.environ["RTN_REV_CHUNK"]
    # 70,000 nodes in two equal chunks of 35,000
    idx = np.unique(np.concatenate([np.arange(0, 70000, 997), np.arange(34995, 35005), [69999]]))
    f, j, _ = om.batched_eval(z[idx], 1)
    assert max_node_rel_error(got.jacobians[idx], j) < 1e-3
    assert max_node_rel_error(got.values[idx], f) < 1e-3
    ef, ej, _ = _errs(_net([17] + [512] * 12 + [6], "silu", 2.5), 2048)
    assert ef < 5e-3 and ej < 5e-3, (ef, ej)


def test_reverse_matches_forward_mode_and_bitwise_rows():
    """Reverse and forward mode agree within TF32 (same values: f comes from the same
    value path); reverse-mode rows of a batch are bit-identical to single-node calls."""
    om = _net([17] + [512] * 6 + [6], "silu", 2.0)
    z = quad_nodes(9, 2000)
    pm = to_product_model(om)
    fwd = pm.engine().prepare(z, 1)
    eng = pm.engine(jacobian_mode=1)
    rev = eng.prepare(z, 1)
    assert max_node_rel_error(rev.jacobians, fwd.jacobians) < 1e-3
    for i in (0, 127, 128, 255, 1999):
        one = eng.prepare(z[i:i + 1], 1)
        assert np.array_equal(one.values[0], rev.values[i]) and np.array_equal(one.jacobians[0], rev.jacobians[i])


def test_jacobian_mode_api_errors_and_switching():
    L = _lib.lib()
    om = _net([17] + [512] * 3 + [6], "silu", 1.5)
    eng = to_product_model(om).engine()
    assert L.rtn_ctx_set_jacobian_mode(eng.ctx_ptr, 2) == _lib.RTN_ECONFIG
    z = quad_nodes(4, 300)
    a = eng.prepare(z, 1)
    raise_for_status(L.rtn_ctx_set_jacobian_mode(eng.ctx_ptr, 1))
    b = eng.prepare(z, 1)
    raise_for_status(L.rtn_ctx_set_jacobian_mode(eng.ctx_ptr, 0))
    c = eng.prepare(z, 1)
    assert np.array_equal(a.jacobians, c.jacobians) and not np.array_equal(a.jacobians, b.jacobians)
    # order 2 calls keep forward mode; unsupported models refuse reverse mode
    raise_for_status(L.rtn_ctx_set_jacobian_mode(eng.ctx_ptr, 1))
    h = eng.prepare(z[:5], 2)
    assert np.isfinite(h.hessians).all()
    for sizes, prec in (([17] + [256] * 3 + [6], "tf32"), ([17] + [512] * 3 + [3], "3xtf32"),
                        ([30, 512, 512, 6], "tf32"), ([17] + [512] * 3 + [6], "bf16")):
        e2 = to_product_model(_net(sizes, "silu", 1.0)).engine(precision=_lib.PRECISIONS[prec])
        assert L.rtn_ctx_set_jacobian_mode(e2.ctx_ptr, 1) == _lib.RTN_EUNSUPPORTED, (sizes, prec)


def test_reverse_mode_latency_graphs_follow_the_mode():
    """Latency-mode contexts capture graphs; switching the Jacobian mode drops them."""
    L = _lib.lib()
    om = _net([17] + [512] * 3 + [6], "silu", 1.5)
    pm = to_product_model(om)
    eng = pm.engine(latency_mode=1)
    z = quad_nodes(6, 20)
    a = eng.prepare(z, 1)
    raise_for_status(L.rtn_ctx_set_jacobian_mode(eng.ctx_ptr, 1))
    b = eng.prepare(z, 1)
    ref = pm.engine(jacobian_mode=1).prepare(z, 1)
    assert np.array_equal(b.jacobians, ref.jacobians)
    f, j, _ = om.batched_eval(z, 1)
    assert max_node_rel_error(a.jacobians, j) < 1e-3 and max_node_rel_error(b.jacobians, j) < 1e-3


@pytest.mark.parametrize("prec,bound", [("3xtf32", 1e-5), ("bf16x3", 1e-4)])
@pytest.mark.parametrize("width,depth,k", [(512, 12, 600), (256, 5, 2000), (512, 3, 97)])
def test_reverse_mode_split_precision_on_pair_tiles(prec, bound, width, depth, k):
    """3xTF32 / bf16x3 reverse mode (the pair kernel's value and adjoint variants,
    fp32 slope scratch) on the conditioned nets of the forward-mode precision tests,
    at the modes' bounds; ragged K and more nodes than one tile per CTA pair."""
    om = _net([17] + [width] * depth + [6], "silu", 2.5 if depth == 12 else 2.0)
    z = quad_nodes(13, k)
    got = to_product_model(om).engine(precision=_lib.PRECISIONS[prec], jacobian_mode=1).prepare(z, 1)
    f, j, _ = om.batched_eval(z, 1)
    ef, ej = max_node_rel_error(got.values, f), max_node_rel_error(got.jacobians, j)
    assert ef < bound and ej < bound, (prec, width, depth, ef, ej)


@pytest.mark.parametrize("prec", ["3xtf32", "bf16x3"])
def test_reverse_pair_chunking_is_bitwise_neutral(prec):
    """Scratch chunking of the pair-kernel reverse passes (forced small by
    RTN_REV_CHUNK: 7 equal chunks of 286 nodes) gives the same bits as one chunk."""
    om = _net([17] + [256] * 5 + [6], "silu", 2.0)
    z = quad_nodes(17, 2000)
    pm = to_product_model(om)
    one = pm.engine(precision=_lib.PRECISIONS[prec], jacobian_mode=1).prepare(z, 1)
    os.environ["RTN_REV_CHUNK"] = "300"
    try:
        many = pm.engine(precision=_lib.PRECISIONS[prec], jacobian_mode=1).prepare(z, 1)
    finally:
        del os.environ["RTN_REV_CHUNK"]
    assert np.array_equal(one.values, many.values) and np.array_equal(one.jacobians, many.jacobians)


@pytest.mark.parametrize("prec,bound", [("3xtf32", 1e-5), ("bf16x3", 1e-4)])
@pytest.mark.parametrize("n_in,width", [(3, 256), (24, 256), (9, 512), (24, 512)])
def test_reverse_pair_input_widths(prec, bound, n_in, width):
    """Pair-kernel reverse passes at the input widths the adjoint's 32-column W0'
    output covers (n_in <= 24), both padded widths, 6 outputs; ragged K."""
    om = _net([n_in] + [width] * 4 + [6], "silu", 2.0)
    z = _z(n_in, 333, n_in)
    got = to_product_model(om).engine(precision=_lib.PRECISIONS[prec], jacobian_mode=1).prepare(z, 1)
    f, j, _ = om.batched_eval(z, 1)
    ef, ej = max_node_rel_error(got.values, f), max_node_rel_error(got.jacobians, j)
    assert ef < bound and ej < bound, (prec, n_in, width, ef, ej)


@pytest.mark.parametrize("prec", ["tf32", "3xtf32", "bf16x3"])
def test_reverse_empty_and_single_node(prec):
    """K = 0 launches nothing and returns empty blocks; K = 1 matches the oracle
    (the reference's single-input contract, proj/src/neural.cpp:300-318)."""
    om = _net([17] + [512] * 3 + [6], "silu", 2.0)
    eng = to_product_model(om).engine(precision=_lib.PRECISIONS[prec], jacobian_mode=1)
    z = quad_nodes(3, 1)
    empty = eng.prepare(z[:0], 1)
    assert empty.values.shape == (0, 6) and empty.jacobians.shape == (0, 6, 17)
    one = eng.prepare(z, 1)
    f, j, _ = om.batched_eval(z, 1)
    bound = 1e-5 if prec == "3xtf32" else 1e-3
    assert max_node_rel_error(one.values, f) < bound and max_node_rel_error(one.jacobians, j) < bound
