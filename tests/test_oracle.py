"""CPU tests: the oracle (oracle/, test infrastructure) pinned against the
reference's own known-answer / finite-difference tests, and the committed
golden fixtures reproduced from it."""
import json
import os
import subprocess

import numpy as np
import pytest

import oracle

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def test_reference_test_suite_restated(oracle_lib):
    """oracle/test_oracle.cpp re-expresses proj/tests/test_neural.cpp:11-152,231-282
    and proj/tests/test_taylor.cpp:8-135 (same seeds, shapes, tolerances)."""
    r = subprocess.run([oracle.TEST_BIN], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_single_linear_layer_known_answer(oracle_lib):
    # proj/tests/test_neural.cpp:11-20
    om = oracle.OracleModel.make_mlp([3, 2], "tanh", 1)
    w = np.array([[1.0, -2.0, 0.5], [0.0, 3.0, 1.0]])
    b = np.array([0.25, -1.0])
    om.set_layer(0, w, b)
    z = np.array([[0.3, -0.7, 2.0]])
    f, j, _ = om.batched_eval(z, 1)
    assert np.max(np.abs(f[0] - (w @ z[0] + b))) < 1e-15
    assert np.array_equal(j[0], w)


def test_closed_form_hessian(oracle_lib):
    # proj/tests/test_neural.cpp:76-89 (tanh) and the SiLU analogue
    for act in ("tanh", "silu"):
        om = oracle.OracleModel.make_mlp([1, 1, 1], act, 4)
        om.set_layer(0, np.array([[0.8]]), np.array([-0.3]))
        om.set_layer(1, np.array([[1.7]]), np.array([0.0]))
        pre = 0.8 * 0.45 - 0.3
        if act == "tanh":
            t = np.tanh(pre)
            spp = -2 * t * (1 - t * t)
        else:
            s = 1 / (1 + np.exp(-pre))
            spp = s * (1 - s) * (2 + pre * (1 - 2 * s))
        _, _, h = om.batched_eval(np.array([[0.45]]), 2)
        assert abs(h[0, 0, 0, 0] - 1.7 * 0.8 * 0.8 * spp) <= 1e-12


def test_forward_mode_matches_reverse_mode(oracle_lib):
    """The GPU algorithm (forward-mode tangents) agrees with the reference's
    reverse sweep to fp64 rounding on the quadrotor shape."""
    for act in ("tanh", "silu"):
        om = oracle.OracleModel.random_net([17, 64, 64, 64, 6], act, 3, True)
        z = oracle.quad_nodes(9, 16)
        f, j, h = om.batched_eval(z, 2)
        f2, j2, h2 = om.forward_mode(z, 2)
        assert oracle.rel_error(f2, f) < 1e-13
        assert oracle.rel_error(j2, j) < 1e-13
        assert oracle.rel_error(h2, h) < 1e-12


def test_batch_equals_single_bitwise(oracle_lib):
    # proj/tests/test_neural.cpp:119-145 contract at the quadrotor shape
    om = oracle.OracleModel.random_net([17, 32, 32, 6], "silu", 23, True)
    z = oracle.quad_nodes(4, 13)
    f, j, _ = om.batched_eval(z, 1, threads=4)
    for i in range(13):
        fi, ji, _ = om.batched_eval(z[i:i + 1], 1, threads=1)
        assert np.array_equal(fi[0], f[i]) and np.array_equal(ji[0], j[i])


@pytest.mark.parametrize("name", ["cfg1_tanh_2x64_N10", "silu_3x128_N8", "tanh_6_32_32_4_K13"])
def test_golden_fixture_reproduced(oracle_lib, name):
    rec = json.load(open(os.path.join(GOLDEN, name + ".json")))
    om = oracle.OracleModel.load(os.path.join(GOLDEN, rec["model_file"]))
    z = np.array(rec["z"])
    f, j, h = om.batched_eval(z, rec["order"])
    assert np.array_equal(f, np.array(rec["f"]))
    assert np.array_equal(j, np.array(rec["jac"]))
    if rec["order"] == 2:
        assert np.array_equal(h, np.array(rec["hess"]))


def test_golden_fd_consistency(oracle_lib):
    """Fixture Jacobians agree with central differences of the fixture model
    (proj/tests/test_neural.cpp:45-57 style), so the fixtures are not just
    self-consistent."""
    rec = json.load(open(os.path.join(GOLDEN, "cfg1_tanh_2x64_N10.json")))
    om = oracle.OracleModel.load(os.path.join(GOLDEN, rec["model_file"]))
    z = np.array(rec["z"])
    j = np.array(rec["jac"])
    h = 1e-5
    for i in range(z.shape[0]):
        fd = np.zeros_like(j[i])
        for k in range(z.shape[1]):
            zp, zm = z[i].copy(), z[i].copy()
            zp[k] += h
            zm[k] -= h
            fp, _, _ = om.batched_eval(zp[None], 0)
            fm, _, _ = om.batched_eval(zm[None], 0)
            fd[:, k] = (fp[0] - fm[0]) / (2 * h)
        assert oracle.rel_error(j[i], fd) < 1e-7
