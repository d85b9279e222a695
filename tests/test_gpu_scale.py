"""Parity at production batch sizes: every kernel instantiation the chooser
selects for the throughput configs runs many tiles per CTA pair here (cfg5:
200k nodes of 12x512 SiLU through rtn_pair_kernel<512,4,4,80,TF32>, ~340
tiles per pair; cfg4: 81,920 nodes of 5x256 through the rows kernel), on
conditioned nets (|J| ~ 1), and a sample of ~1 in 1000 nodes (plus the first
and last) is checked against the fp64 oracle. Metric as in
proj/tests/oracles.hpp:30-32, per node and block."""
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


def _sampled(om, prec, k, kernel, monkeypatch, every=1000, seed=2203):
    if kernel:
        monkeypatch.setenv("RTN_KERNEL", kernel)
    else:
        monkeypatch.delenv("RTN_KERNEL", raising=False)
    z = oracle.quad_nodes(seed, k)
    got = oracle.to_product_model(om).engine(precision=_lib.PRECISIONS[prec]).prepare(z, 1)
    assert np.isfinite(got.values).all() and np.isfinite(got.jacobians).all()
    idx = np.unique(np.concatenate([np.arange(0, k, every), np.arange(k - 7, k), np.random.default_rng(1).integers(0, k, 64)]))
    f, j, _ = om.batched_eval(z[idx], 1)
    return max(oracle.max_node_rel_error(got.values[idx], f),
               oracle.max_node_rel_error(got.jacobians[idx, :, :13], j[:, :, :13]),
               oracle.max_node_rel_error(got.jacobians[idx, :, 13:], j[:, :, 13:]))


def test_cfg5_headline_kernel_tf32_many_tiles(monkeypatch):
    """The bench's TF32 kernel (chooser default at K >> #SMs: the split kernel), 200,704 nodes."""
    err = _sampled(_net([17] + [512] * 12 + [6], "silu", 2.5), "tf32", 200704, None, monkeypatch)
    assert err < 5e-3, err  # TF32's documented limit on this net (test_gpu_precision.py)
    err = _sampled(_net([17] + [512] * 12 + [6], "silu", 2.0), "tf32", 200704, None, monkeypatch)
    assert err < 1e-3, err


def test_cfg5_shape_3xtf32_many_tiles(monkeypatch):
    """3xTF32 at width 512 (24-row tiles, four main accumulators), 100k nodes."""
    err = _sampled(_net([17] + [512] * 12 + [6], "silu", 2.5), "3xtf32", 100352, None, monkeypatch)
    assert err < 1e-5, err


def test_cfg5_shape_bf16x3_many_tiles(monkeypatch):
    err = _sampled(_net([17] + [512] * 12 + [6], "silu", 2.5), "bf16x3", 100352, None, monkeypatch)
    assert err < 1e-4, err


@pytest.mark.parametrize("prec,bound", [("tf32", 1e-3), ("3xtf32", 1e-5), ("bf16x3", 1e-4)])
def test_cfg4_every_mode_many_tiles(prec, bound, monkeypatch):
    """cfg4 (4096 x 20 nodes, 5x256): rows kernel (TF32) / pair kernel P = 4 (split modes)."""
    err = _sampled(_net([17] + [256] * 5 + [6], "silu", 1.5), prec, 81920, None, monkeypatch, every=500)
    assert err < bound, (prec, err)


def test_width256_pair_kernel_narrow_inputs_many_tiles(monkeypatch):
    """TF32 width 256 with n_in < 7 (the 'a' variant's 3 features) runs the pair
    kernel with P = 16 nodes per CTA side."""
    om = _net([3, 256, 256, 256, 3], "silu", 2.0)
    z = np.random.default_rng(3).uniform(-2, 2, (50000, 3))
    monkeypatch.delenv("RTN_KERNEL", raising=False)
    got = oracle.to_product_model(om).engine().prepare(z, 1)
    idx = np.arange(0, 50000, 97)
    f, j, _ = om.batched_eval(z[idx], 1)
    assert oracle.max_node_rel_error(got.values[idx], f) < 1e-3
    assert oracle.max_node_rel_error(got.jacobians[idx], j) < 1e-3


def test_latency_tiles_forced_on_a_large_batch(monkeypatch):
    """The latency geometry (one node per CTA side) normally sees <= 1 tile per
    pair; forced here onto 3,000 nodes so every pair walks ~20 tiles."""
    err = _sampled(_net([17] + [512] * 6 + [6], "silu", 2.0), "tf32", 3000, "latency", monkeypatch, every=50)
    assert err < 1e-3, err


def test_cfg5_shape_bf16_single_pass_many_tiles(monkeypatch):
    """Single-pass BF16 at cfg5 scale (the rowsb kernel: A in TMEM), 100k nodes, gain 2.0."""
    err = _sampled(_net([17] + [512] * 12 + [6], "silu", 2.0), "bf16", 100352, None, monkeypatch)
    assert err < 1e-3, err


def test_cfg5_pair_kernel_tf32_many_tiles(monkeypatch):
    """The TF32 pair kernel (rtn_pair_kernel<512,4,4,80,TF32>, forced) on the same shape."""
    err = _sampled(_net([17] + [512] * 12 + [6], "silu", 2.0), "tf32", 200704, "pair", monkeypatch)
    assert err < 1e-3, err
