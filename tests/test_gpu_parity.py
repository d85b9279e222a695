"""GPU parity: the sm_100a path (through the C-ABI) against the fp64 oracle.

Tolerance (north star): norm-wise relative error ‖a−b‖∞/(1+‖b‖∞)
(proj/tests/oracles.hpp:30-32) per node and per block (f, A = ∂f/∂x, B =
∂f/∂u), max over nodes: 1e-3 in TF32 mode, 1e-5 in 3xTF32 mode.
"""
import numpy as np
import pytest

import oracle
from oracle import OracleModel, max_node_rel_error, quad_nodes, to_product_model

TF32_TOL = 1e-3

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["pair", "latency", "quad", "rows", "split"])
def kernel(request, monkeypatch):
    """Every device kernel: CTA-pair throughput tiles, CTA-pair latency tiles (P=1), the
    4-CTA-cluster latency kernel (width-512 models, K <= 2·(#SMs/4); others fall back),
    the width-256 rows kernel (activations as the MMA's A operand in TMEM; TF32 width-256
    models with 7 <= n_in <= 31, others fall back) and the width-512 split kernel (A split
    between TMEM and shared memory; TF32 width-512 models with 7 <= n_in <= 31)."""
    monkeypatch.setenv("RTN_KERNEL", request.param)
    return request.param


def _blocks(f, jac):
    return {"f": f, "A": jac[:, :, :13], "B": jac[:, :, 13:]}


def _check(model_sizes, act, k, seed=2203, rng_seed=11, random_norm=True, tol=TF32_TOL):
    from paper_2203_07747_b200 import mlp_batched_eval, EvalOrder
    om = OracleModel.random_net(model_sizes, act, rng_seed, random_norm)
    pm = to_product_model(om)
    z = quad_nodes(seed, k) if model_sizes[0] == 17 else np.random.default_rng(seed).uniform(-2, 2, (k, model_sizes[0]))
    f_ref, j_ref, _ = om.batched_eval(z, 1)
    got = mlp_batched_eval(pm, z, EvalOrder.JACOBIAN)
    ef = max_node_rel_error(got.values, f_ref)
    ej = max_node_rel_error(got.jacobians, j_ref)
    assert np.all(np.isfinite(got.values)) and np.all(np.isfinite(got.jacobians))
    assert ef < tol, f"f rel err {ef}"
    assert ej < tol, f"J rel err {ej}"
    if model_sizes[0] == 17:
        for name, blk in _blocks(got.values, got.jacobians).items():
            ref = _blocks(f_ref, j_ref)[name]
            assert max_node_rel_error(blk, ref) < tol, name
    return ef, ej


def test_cfg1_tanh_2x64():
    _check([17, 64, 64, 6], "tanh", 10)


def test_cfg2_silu_5x256_latency_shape(kernel):
    _check([17] + [256] * 5 + [6], "silu", 20)


def test_cfg3_silu_12x512(kernel):
    _check([17] + [512] * 12 + [6], "silu", 20)


def test_ragged_tile_counts(kernel):
    # K not a multiple of the nodes-per-tile, and more tiles than SMs
    for k in (1, 3, 5, 7, 13, 601):
        _check([17, 128, 128, 6], "silu", k)


def test_reference_shapes_small_nets():
    # the reference's own test shapes (proj/tests/test_neural.cpp, test_taylor.cpp)
    _check([5, 16, 16, 3], "tanh", 20, random_norm=True)
    _check([6, 32, 32, 4], "tanh", 13)
    _check([4, 16, 3], "tanh", 10)
    _check([3, 10, 2], "relu", 20)


def test_batch_rows_equal_single_calls(kernel):
    # neural.hpp:65-67 contract within the device kernel family: a row of a
    # batch is bit-identical to the single-node call.
    from paper_2203_07747_b200 import mlp_batched_eval, mlp_jacobian, mlp_forward, EvalOrder
    om = OracleModel.random_net([17, 256, 256, 256, 6], "silu", 23)
    pm = to_product_model(om)
    z = quad_nodes(5, 13)
    z[12] = z[0]
    b = mlp_batched_eval(pm, z, EvalOrder.JACOBIAN)
    for i in range(13):
        assert np.array_equal(b.values[i], mlp_forward(pm, z[i]))
        assert np.array_equal(b.jacobians[i], mlp_jacobian(pm, z[i]))
    assert np.array_equal(b.values[0], b.values[12])


def test_throughput_shape_cfg4_subset(kernel):
    _check([17] + [256] * 5 + [6], "silu", 4096)


def test_quad_latency_kernel_ragged_and_bitwise(monkeypatch):
    """4-CTA-cluster latency kernel (csrc/rtn_quad.cuh): odd K (a half-empty
    cluster), the K limit (74 on 148 SMs), and rows of a batch bit-identical to
    single-node calls."""
    from paper_2203_07747_b200 import mlp_batched_eval, EvalOrder
    monkeypatch.setenv("RTN_KERNEL", "quad")
    for k in (1, 2, 3, 5, 73, 74):
        _check([17, 512, 512, 512, 6], "silu", k)
    om = OracleModel.random_net([17] + [512] * 4 + [6], "tanh", 29)
    pm = to_product_model(om)
    z = quad_nodes(8, 9)
    full = mlp_batched_eval(pm, z, EvalOrder.JACOBIAN)
    for i in (0, 4, 8):
        one = mlp_batched_eval(pm, z[i:i + 1], EvalOrder.JACOBIAN)
        assert np.array_equal(one.values[0], full.values[i]) and np.array_equal(one.jacobians[0], full.jacobians[i])


def test_rows_kernel_input_widths_and_ragged_tiles(monkeypatch):
    """rtn_rows.cuh: R = 1 + n_in rows per node, 128 // R nodes per CTA — the
    quadrotor 'full' (17 → 7 nodes), 'a_u' (7 → 16), 'ground' (26 → 4) and the
    widest supported input (31 → 4); K around the tile size (2·NPC per pair),
    one node, and more tiles than CTA pairs; hidden widths below 256 (zero padding)."""
    monkeypatch.setenv("RTN_KERNEL", "rows")
    for k in (1, 13, 14, 15, 4099):
        _check([17] + [256] * 5 + [6], "silu", k)
    _check([7, 256, 256, 3], "silu", 777)
    _check([26, 256, 192, 3], "silu", 1000)
    _check([31, 100, 256, 256, 6], "tanh", 501)
    _check([17, 256, 6], "relu", 300)  # one hidden layer: no MMA layer before the output
    _check([17] + [256] * 12 + [6], "silu", 2000)  # 11 hidden->hidden layers: the bias-table capacity
    _check([17] + [256] * 13 + [6], "silu", 500)   # one more: falls back to the pair kernel


def test_rows_kernel_default_for_width256_throughput(monkeypatch):
    """Without RTN_KERNEL a TF32 width-256 batch above the latency regime runs the
    rows kernel; its rows are bit-identical to single-node calls forced onto it."""
    from paper_2203_07747_b200 import mlp_batched_eval, EvalOrder
    om = OracleModel.random_net([17] + [256] * 5 + [6], "silu", 37)
    z = quad_nodes(6, 3000)
    monkeypatch.delenv("RTN_KERNEL", raising=False)
    full = mlp_batched_eval(to_product_model(om), z, EvalOrder.JACOBIAN)
    f, j, _ = om.batched_eval(z, 1)
    assert max_node_rel_error(full.values, f) < TF32_TOL and max_node_rel_error(full.jacobians, j) < TF32_TOL
    monkeypatch.setenv("RTN_KERNEL", "rows")
    for i in (0, 6, 7, 13, 2999):
        one = mlp_batched_eval(to_product_model(om), z[i:i + 1], EvalOrder.JACOBIAN)
        assert np.array_equal(one.values[0], full.values[i]) and np.array_equal(one.jacobians[0], full.jacobians[i])


def test_quad_kernel_bf16x3_bitwise_and_ragged(monkeypatch):
    """bf16x3 on the 4-CTA latency kernel: ragged K up to the cluster limit within
    the bf16 class tolerance, and rows of a batch bit-identical to single-node calls."""
    from paper_2203_07747_b200 import mlp_batched_eval, EvalOrder
    from paper_2203_07747_b200 import _lib
    monkeypatch.setenv("RTN_KERNEL", "quad")
    om = OracleModel.random_net([17, 512, 512, 512, 6], "silu", 41, True)
    eng = to_product_model(om).engine(precision=_lib.PRECISIONS["bf16x3"])
    for k in (1, 2, 5, 74):
        z = quad_nodes(9, k)
        f, j, _ = om.batched_eval(z, 1)
        got = eng.prepare(z, 1)
        assert max_node_rel_error(got.values, f) < 1e-4 and max_node_rel_error(got.jacobians, j) < 1e-4, k
    z = quad_nodes(10, 7)
    full = eng.prepare(z, 1)
    for i in (0, 3, 6):
        one = eng.prepare(z[i:i + 1], 1)
        assert np.array_equal(one.values[0], full.values[i]) and np.array_equal(one.jacobians[0], full.jacobians[i])


def test_split_kernel_input_widths_and_ragged_tiles(monkeypatch):
    """rtn_split.cuh: R = 1 + n_in rows per node, 128 // R nodes per CTA — 17 (7
    nodes), 15 (8: the largest node count whose next-tile layer-0 tables are
    precomputed), 7 (16: tables per quarter at the tile boundary), 26 and 31 (4);
    K around the tile size and above the CTA-pair count; hidden widths that pad to
    512; 1 to 4 hidden->hidden layers (the precomputed tables are spread over the
    first four layers' idle windows; shorter nets finish them at the tile boundary)."""
    monkeypatch.setenv("RTN_KERNEL", "split")
    for k in (1, 13, 14, 15, 4099):
        _check([17] + [512] * 4 + [6], "silu", k)
    _check([15, 512, 512, 512, 6], "silu", 2500)
    _check([7, 512, 512, 3], "silu", 3000)
    _check([26, 512, 300, 3], "silu", 1000)
    _check([31, 400, 512, 512, 6], "tanh", 501)
    _check([17, 512, 6], "relu", 2100)             # one hidden layer: layer 0 straight into the output layer
    _check([17, 512, 512, 6], "silu", 2100)        # one hidden->hidden layer
    _check([17] + [512] * 4 + [6], "tanh", 2100)   # three
    _check([17] + [512] * 5 + [6], "silu", 2100)   # four


def test_split_kernel_default_and_bitwise_rows(monkeypatch):
    """Without RTN_KERNEL a TF32 width-512 batch above the latency regime runs the
    split kernel; its rows are bit-identical to single-node calls forced onto it."""
    from paper_2203_07747_b200 import mlp_batched_eval, EvalOrder
    om = OracleModel.random_net([17] + [512] * 6 + [6], "silu", 41)
    z = quad_nodes(9, 5000)
    monkeypatch.delenv("RTN_KERNEL", raising=False)
    full = mlp_batched_eval(to_product_model(om), z, EvalOrder.JACOBIAN)
    f, j, _ = om.batched_eval(z, 1)
    assert max_node_rel_error(full.values, f) < TF32_TOL and max_node_rel_error(full.jacobians, j) < TF32_TOL
    monkeypatch.setenv("RTN_KERNEL", "split")
    for i in (0, 6, 7, 13, 14, 2072, 4999):
        one = mlp_batched_eval(to_product_model(om), z[i:i + 1], EvalOrder.JACOBIAN)
        assert np.array_equal(one.values[0], full.values[i]) and np.array_equal(one.jacobians[0], full.jacobians[i])


def test_rowsb_kernel_bf16_widths_ragged_and_bitwise(monkeypatch):
    """rtn_rowsb.cuh (BF16, width 512, the whole layer input as the A operand in
    TMEM): equal to the pair kernel's BF16 results within the bf16 class on the
    input widths it takes (15, 17, 26, 31), ragged K, 1 to 5 hidden->hidden
    layers, and rows of a batch bit-identical to single-node calls."""
    from paper_2203_07747_b200 import _lib
    bf16 = _lib.PRECISIONS["bf16"]

    def run(sizes, act, k, kernel, seed=2203):
        om = OracleModel.random_net(sizes, act, 11, True)
        monkeypatch.setenv("RTN_KERNEL", kernel)
        z = quad_nodes(seed, k) if sizes[0] == 17 else np.random.default_rng(seed).uniform(-2, 2, (k, sizes[0]))
        got = to_product_model(om).engine(precision=bf16).prepare(z, 1)
        f, j, _ = om.batched_eval(z, 1)
        return got, max(max_node_rel_error(got.values, f), max_node_rel_error(got.jacobians, j))

    for sizes, act, k in (([17] + [512] * 4 + [6], "silu", 1), ([17] + [512] * 4 + [6], "silu", 15),
                          ([17] + [512] * 4 + [6], "silu", 4099), ([15, 512, 512, 512, 6], "silu", 2500),
                          ([26, 512, 300, 3], "silu", 1000), ([31, 400, 512, 512, 6], "tanh", 501),
                          ([17, 512, 6], "relu", 2100), ([17] + [512] * 6 + [6], "silu", 2100)):
        got, err = run(sizes, act, k, "rowsb")
        ref, err_pair = run(sizes, act, k, "pair")
        assert np.isfinite(got.values).all() and np.isfinite(got.jacobians).all()
        assert err < max(2 * err_pair, 2e-3), (sizes, k, err, err_pair)
    om = OracleModel.random_net([17] + [512] * 6 + [6], "silu", 41)
    z = quad_nodes(9, 3000)
    monkeypatch.setenv("RTN_KERNEL", "rowsb")
    eng = to_product_model(om).engine(precision=bf16)
    full = eng.prepare(z, 1)
    for i in (0, 6, 7, 13, 14, 2999):
        one = eng.prepare(z[i:i + 1], 1)
        assert np.array_equal(one.values[0], full.values[i]) and np.array_equal(one.jacobians[0], full.jacobians[i])
