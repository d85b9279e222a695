"""CPU tests of the product's host-side logic: model construction, RMLP files,
synthetic generators, validation errors and FLOP accounting. No GPU calls."""
import os

import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import (ConfigError, MlpModel, flops_per_node, load_model, make_mlp, parse_arch,
                                   save_model, synth_quad_nodes)
from paper_2203_07747_b200.taylor import TaylorApprox, eval_taylor, eval_taylor_jacobian


def test_make_mlp_matches_reference_init(oracle_lib):
    """MakeMlp semantics (proj/src/neural.cpp:465-489): same mt19937_64 draws."""
    for sizes, seed in (([17, 64, 64, 6], 2064), ([17] + [256] * 5 + [6], 5256), ([3, 2], 7)):
        m = make_mlp(sizes, "silu", "full", seed)
        om = oracle.OracleModel.make_mlp(sizes, "silu", seed)
        for (w, b), pw, pb in zip(om.layers(), m.weights, m.biases):
            assert np.array_equal(w, pw) and np.array_equal(b, pb)


def test_synthetic_nodes_match_oracle(oracle_lib):
    assert np.array_equal(synth_quad_nodes(2203, 257), oracle.quad_nodes(2203, 257))
    z = synth_quad_nodes(1, 100)
    assert np.allclose(np.linalg.norm(z[:, 3:7], axis=1), 1.0)  # unit quaternions
    assert np.all((z[:, 13:] >= 0.5) & (z[:, 13:] <= 5.0))


@pytest.mark.parametrize("act", ["tanh", "relu", "silu"])
def test_rmlp_round_trip_and_interop(tmp_path, oracle_lib, act):
    """RMLP v1 (tanh/relu, proj/src/neural.cpp:685-755) and v2 (SiLU): python
    writer → oracle reader and oracle writer → python reader, bit-exact."""
    om = oracle.OracleModel.random_net([7, 10, 3], act, 55, True)
    p1 = str(tmp_path / "o.rmlp")
    om.save(p1)
    m = load_model(p1)
    assert m.activation == act and m.layer_sizes == [7, 10, 3]
    for (w, b), pw, pb in zip(om.layers(), m.weights, m.biases):
        assert np.array_equal(w, pw) and np.array_equal(b, pb)
    p2 = str(tmp_path / "p.rmlp")
    save_model(m, p2)
    assert os.path.exists(p2 + ".json")
    om2 = oracle.OracleModel.load(p2)
    for (w, b), (w2, b2) in zip(om.layers(), om2.layers()):
        assert np.array_equal(w, w2) and np.array_equal(b, b2)
    for a, b in zip(om.norm(), om2.norm()):
        assert np.array_equal(a, b)
    with open(p2, "rb") as fh:
        head = fh.read(9)
    assert head[:4] == b"RMLP" and head[4] == (2 if act == "silu" else 1)


def test_v1_reader_tag_semantics(tmp_path):
    """A v1 file's activation byte: 0 → tanh, anything else → relu (neural.cpp:729)."""
    m = make_mlp([3, 4, 2], "relu", "full", 1)
    p = str(tmp_path / "r.rmlp")
    save_model(m, p)
    data = bytearray(open(p, "rb").read())
    data[8] = 7
    open(p, "wb").write(bytes(data))
    assert load_model(p).activation == "relu"


def test_validation_errors():
    m = make_mlp([4, 8, 2], "tanh", "full", 0)
    m.in_scale = np.array([1.0, 0.0, 1.0, 1.0])
    with pytest.raises(ConfigError):
        m.validate()
    with pytest.raises(ConfigError):
        make_mlp([4], "tanh")
    with pytest.raises(ConfigError):
        load_model("/nonexistent/model.rmlp")
    bad = MlpModel([3, 2], [np.zeros((2, 2))], [np.zeros(2)], "tanh", "full", np.zeros(3), np.ones(3),
                   np.zeros(2), np.ones(2))
    with pytest.raises(ConfigError):
        bad.validate()


def test_parse_arch():
    # proj/tests/test_neural.cpp:277-282
    assert parse_arch("3x32") == [32, 32, 32]
    assert parse_arch("18,18") == [18, 18]
    assert parse_arch("64") == [64]
    with pytest.raises(ConfigError):
        parse_arch("0x4")


def test_parameter_count_and_flops():
    m = make_mlp([17] + [512] * 12 + [6], "silu", "full", 12512)
    assert m.parameter_count() == 2901510          # SURVEY §6 note
    assert m.arch_name() == "N-12-512"
    # BASELINE.md §2 table
    assert flops_per_node([17, 64, 64, 6]) == 200448
    assert flops_per_node([17] + [256] * 5 + [6]) == 9649152
    assert flops_per_node([17] + [512] * 12 + [6]) == 104232960
    assert flops_per_node([17] + [512] * 12 + [6], 2) == 2 * (1 + 17 + 153) * 2895360


def test_taylor_consumers_match_oracle(oracle_lib):
    """Host-side EvalTaylor / EvalTaylorJacobian (proj/src/taylor.cpp:57-74)."""
    rng = np.random.default_rng(0)
    om = oracle.OracleModel.random_net([3, 14, 2], "tanh", 5, True)
    z0 = rng.uniform(-1, 1, (1, 3))
    f, j, h = om.batched_eval(z0, 2)
    a = TaylorApprox(0, 2, z0[0], f[0], j[0], [h[0, o] for o in range(2)])
    a.validate()
    assert np.array_equal(eval_taylor(a, z0[0]), f[0])           # expansion point exact
    assert np.array_equal(eval_taylor_jacobian(a, z0[0]), j[0])
    z = z0[0] + 0.3 * rng.uniform(-1, 1, 3)
    y = eval_taylor(a, z)
    dz = z - z0[0]
    ref = f[0] + j[0] @ dz + 0.5 * np.array([dz @ h[0, o] @ dz for o in range(2)])
    assert np.allclose(y, ref, rtol=0, atol=1e-14)
    with pytest.raises(ConfigError):
        TaylorApprox(0, 2, z0[0], f[0], j[0], []).validate()


def test_make_zero_network():
    """proj/src/bench.cpp:25-36: MakeMlp (tanh) hidden layers, last layer zeroed;
    positive dimensions required."""
    from paper_2203_07747_b200 import ConfigError, make_mlp, make_zero_network
    z = make_zero_network(3, 32, 17, 6, 3032)
    m = make_mlp([17, 32, 32, 32, 6], "tanh", "full", 3032)
    assert z.layer_sizes == [17, 32, 32, 32, 6] and z.activation == "tanh"
    for l in range(3):
        assert np.array_equal(z.weights[l], m.weights[l]) and np.array_equal(z.biases[l], m.biases[l])
    assert not z.weights[-1].any() and not z.biases[-1].any()
    for bad in ((0, 32, 17, 6), (3, 0, 17, 6), (3, 32, 0, 6), (3, 32, 17, 0)):
        with pytest.raises(ConfigError):
            make_zero_network(*bad, 1)
