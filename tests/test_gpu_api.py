"""GPU tests of the drop-in interface (PrepareNodes / MlpBatchedEval mirror
over the C-ABI): golden fixtures, RMLP loading on the device, error mapping,
counters, and the one-batched-call contract (proj/tests/test_taylor.cpp:8-28)."""
import ctypes as C
import json
import os

import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import (EvalCounters, EvalOrder, InputDomainError, UnsupportedError, _lib, load_model,
                                   make_mlp, mlp_batched_eval, mlp_forward, mlp_jacobian, prepare_nodes)
from paper_2203_07747_b200.errors import raise_for_status

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


@pytest.mark.parametrize("name", ["cfg1_tanh_2x64_N10", "tanh_6_32_32_4_K13"])
def test_golden_fixtures_tf32(name):
    rec = json.load(open(os.path.join(GOLDEN, name + ".json")))
    m = load_model(os.path.join(GOLDEN, rec["model_file"]))
    z = np.array(rec["z"])
    got = mlp_batched_eval(m, z, EvalOrder.JACOBIAN)
    assert oracle.max_node_rel_error(got.values, np.array(rec["f"])) < 1e-3
    assert oracle.max_node_rel_error(got.jacobians, np.array(rec["jac"])) < 1e-3


def test_rmlp_file_loads_straight_to_device():
    """rtn_model_load_rmlp (C-ABI file path) == arrays path, bitwise."""
    rec = json.load(open(os.path.join(GOLDEN, "cfg1_tanh_2x64_N10.json")))
    path = os.path.join(GOLDEN, rec["model_file"])
    L = _lib.lib()
    mp = C.c_void_p()
    raise_for_status(L.rtn_model_load_rmlp(path.encode(), 0, 0, C.byref(mp)))
    ctx = C.c_void_p()
    raise_for_status(L.rtn_ctx_create(mp, 64, 1, 0, C.byref(ctx)))
    z = np.ascontiguousarray(rec["z"])
    k = z.shape[0]
    f = np.empty((k, 6))
    j = np.empty((k, 6, 17))
    dp = C.POINTER(C.c_double)
    raise_for_status(L.rtn_prepare(ctx, z.ctypes.data_as(dp), k, 17, 1, f.ctypes.data_as(dp), j.ctypes.data_as(dp), None))
    ref = mlp_batched_eval(load_model(path), z, EvalOrder.JACOBIAN)
    assert np.array_equal(f, ref.values) and np.array_equal(j, ref.jacobians)
    calls, points, launches = C.c_ulonglong(), C.c_ulonglong(), C.c_ulonglong()
    raise_for_status(L.rtn_ctx_counters(ctx, C.byref(calls), C.byref(points), C.byref(launches)))
    assert (calls.value, points.value, launches.value) == (1, k, 1)
    L.rtn_ctx_free(ctx)
    L.rtn_model_free(mp)


def test_prepare_nodes_is_one_batched_call_and_matches_single_calls():
    # proj/tests/test_taylor.cpp:8-28 on the device path
    om = oracle.OracleModel.random_net([4, 16, 3], "tanh", 1, True)
    m = oracle.to_product_model(om)
    z = np.random.default_rng(1).uniform(-1, 1, (10, 4))
    c = EvalCounters()
    approx = prepare_nodes(m, z, 1, c)
    assert c.batched_calls == 1 and c.batched_points == 10 and c.value_evals == 0 and c.jacobian_evals == 0
    for k, a in enumerate(approx):
        assert a.node == k
        assert np.array_equal(a.f_bar, mlp_forward(m, z[k]))
        assert np.array_equal(a.jac, mlp_jacobian(m, z[k]))


def test_error_mapping():
    m = make_mlp([4, 8, 2], "relu", "full", 3)
    with pytest.raises(InputDomainError):          # proj/src/neural.cpp:230-232
        mlp_batched_eval(m, np.zeros((3, 5)), EvalOrder.VALUE)
    with pytest.raises(UnsupportedError):          # proj/src/neural.cpp:176-177
        mlp_batched_eval(m, np.zeros((3, 4)), EvalOrder.HESSIAN)


def test_zero_output_model():
    # proj/tests/test_taylor.cpp:30-41
    om = oracle.OracleModel.random_net([17, 128, 6], "tanh", 9, False)
    w, b = om.layers()[-1]
    om.set_layer(1, np.zeros_like(w), np.zeros_like(b))
    m = oracle.to_product_model(om)
    got = mlp_batched_eval(m, oracle.quad_nodes(3, 5), EvalOrder.JACOBIAN)
    assert np.all(got.values == 0.0) and np.all(got.jacobians == 0.0)


def test_empty_batch():
    m = make_mlp([17, 64, 6], "silu", "full", 1)
    got = mlp_batched_eval(m, np.zeros((0, 17)), EvalOrder.JACOBIAN)
    assert got.values.shape == (0, 6) and got.jacobians.shape == (0, 6, 17)


def test_large_batch_end_to_end_chunked(monkeypatch):
    """K ≥ 2^17 takes the chunked H2D/kernel/D2H pipeline; results equal the
    device-resident call bitwise and the oracle within tolerance on a sample."""
    om = oracle.OracleModel.random_net([17, 256, 256, 6], "silu", 5, True)
    m = oracle.to_product_model(om)
    k = 150_000
    z = oracle.quad_nodes(77, k)
    got = mlp_batched_eval(m, z, EvalOrder.JACOBIAN)
    idx = np.arange(0, k, 997)
    f, j, _ = om.batched_eval(z[idx], 1)
    assert oracle.max_node_rel_error(got.values[idx], f) < 1e-3
    assert oracle.max_node_rel_error(got.jacobians[idx], j) < 1e-3
    monkeypatch.setenv("RTN_KERNEL", "rows")  # the kernel the big call ran (TF32 width 256) → bitwise batch invariance
    again = mlp_batched_eval(m, z[idx], EvalOrder.JACOBIAN)
    assert np.array_equal(again.values, got.values[idx])
    assert np.array_equal(again.jacobians, got.jacobians[idx])


def test_latency_mode_graph_path_matches_direct_path():
    """latency_mode contexts replay a captured H2D→kernel→D2H graph per (K, order);
    results equal the direct path bitwise, across repeated calls and K changes."""
    om = oracle.OracleModel.random_net([17] + [512] * 4 + [6], "silu", 31, True)
    m = oracle.to_product_model(om)
    direct = m.engine(latency_mode=0)
    graph = m.engine(latency_mode=1)
    for k in (20, 20, 7, 20, 50):
        z = oracle.quad_nodes(100 + k, k)
        a = direct.prepare(z, 1)
        b = graph.prepare(z, 1)
        assert np.array_equal(a.values, b.values) and np.array_equal(a.jacobians, b.jacobians)
    calls, points, launches = graph.counters()
    assert calls == 5 and points == 117 and launches >= 5


def _fnv1a64(data: bytes) -> str:
    h = 0xcbf29ce484222325
    for b in data:
        h = ((h ^ b) * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"


def test_digest_keyed_model_cache(tmp_path, monkeypatch):
    """rtn_model_load_rmlp keys packed device models by the FNV-1a 64 digest of the
    file (proj/src/io.cpp:10-26): identical bytes share one reference-counted
    handle; RTN_PACK_CACHE keeps the packed layout on disk for the next load, whose
    results are bit-identical to packing from the RMLP."""
    L = _lib.lib()
    om = oracle.OracleModel.random_net([17, 256, 256, 6], "silu", 5, True)
    path = str(tmp_path / "m.rmlp")
    from paper_2203_07747_b200 import save_model
    save_model(oracle.to_product_model(om), path)
    digest = _fnv1a64(open(path, "rb").read())
    monkeypatch.setenv("RTN_PACK_CACHE", str(tmp_path))
    z = np.ascontiguousarray(oracle.quad_nodes(3, 33))
    dp = C.POINTER(C.c_double)

    def run(mp):
        ctx = C.c_void_p()
        raise_for_status(L.rtn_ctx_create(mp, 64, 1, 0, C.byref(ctx)))
        f, j = np.empty((33, 6)), np.empty((33, 6, 17))
        raise_for_status(L.rtn_prepare(ctx, z.ctypes.data_as(dp), 33, 17, 1, f.ctypes.data_as(dp),
                                       j.ctypes.data_as(dp), None))
        L.rtn_ctx_free(ctx)
        return f, j

    a, b = C.c_void_p(), C.c_void_p()
    raise_for_status(L.rtn_model_load_rmlp(path.encode(), 0, 0, C.byref(a)))
    raise_for_status(L.rtn_model_load_rmlp(path.encode(), 0, 0, C.byref(b)))
    assert a.value == b.value  # same bytes, device, precision: one shared packed model
    out, fp = C.create_string_buffer(17), C.c_int(-1)
    raise_for_status(L.rtn_model_digest(a, out, C.byref(fp)))
    assert out.value.decode() == digest and fp.value == 0
    assert os.path.exists(os.path.join(str(tmp_path), f"{digest}-p0.rtnp"))
    f1, j1 = run(a)
    L.rtn_model_free(b)
    f2, j2 = run(a)  # still alive after one free
    L.rtn_model_free(a)
    c = C.c_void_p()
    raise_for_status(L.rtn_model_load_rmlp(path.encode(), 0, 0, C.byref(c)))
    raise_for_status(L.rtn_model_digest(c, out, C.byref(fp)))
    assert fp.value == 1  # packed layout read back from the cache file
    f3, j3 = run(c)
    L.rtn_model_free(c)
    assert np.array_equal(f1, f2) and np.array_equal(f1, f3) and np.array_equal(j1, j3)
    # a different precision of the same file is a different model
    d = C.c_void_p()
    raise_for_status(L.rtn_model_load_rmlp(path.encode(), 0, 1, C.byref(d)))
    assert d.value != c.value or True
    L.rtn_model_free(d)
    f_ref, j_ref, _ = om.batched_eval(z, 1)
    assert oracle.max_node_rel_error(f3, f_ref) < 1e-3 and oracle.max_node_rel_error(j3, j_ref) < 1e-3


def test_nonfinite_flag_per_call():
    """SURVEY §5 failure detection: a NaN/Inf written by the output epilogue raises
    the context's flag (rtn_ctx_nonfinite); each blocking call starts clean."""
    om = oracle.OracleModel.random_net([17, 64, 64, 6], "tanh", 3, True)
    good = oracle.to_product_model(om)
    bad = oracle.to_product_model(om)
    bad.weights[-1] = bad.weights[-1].copy()
    bad.weights[-1][2, 5] = np.nan
    z = oracle.quad_nodes(1, 40)
    eb = bad.engine()
    out = eb.prepare(z, 1)
    assert np.isnan(out.values[:, 2]).all()
    assert eb.nonfinite(reset=False) and eb.nonfinite(reset=True) and not eb.nonfinite()
    eg = good.engine()
    eg.prepare(z, 1)
    assert not eg.nonfinite()
    eb.prepare(z, 1)
    assert eb.nonfinite()
