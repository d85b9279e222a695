"""CPU tests of the continuity-block builder: the
oracle restatement (oracle/blocks_oracle.cpp) pinned against the reference's
integrator / dynamics / BuildQp tests, and the C-ABI's configuration checks
(same messages as QuadParams::Validate / OcpConfig::Validate) before any device
work."""
import ctypes as C
import re
import subprocess

import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import _lib, qp
from paper_2203_07747_b200.errors import ConfigError, raise_for_status


def test_reference_blocks_tests_restated(oracle_lib):
    """oracle/test_blocks.cpp re-expresses proj/tests/test_integrator.cpp:35-196,
    test_dynamics.cpp:19-134 and test_sqp_rti.cpp:77-128 (same seeds/tolerances)."""
    r = subprocess.run([oracle.TEST_BLOCKS_BIN], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def _quad_case(n_inst, n, seed=3, order=1, sizes=(17, 32, 32, 6)):
    rng = np.random.default_rng(seed)
    xs = np.empty((n_inst, n + 1, 13))
    xs[..., 0:3] = rng.uniform(-2, 2, (n_inst, n + 1, 3))
    q = rng.uniform(-1, 1, (n_inst, n + 1, 4))
    xs[..., 3:7] = q / np.linalg.norm(q, axis=-1, keepdims=True)
    xs[..., 7:10] = rng.uniform(-4, 4, (n_inst, n + 1, 3))
    xs[..., 10:13] = rng.uniform(-3, 3, (n_inst, n + 1, 3))
    us = rng.uniform(0.5, 5.0, (n_inst, n, 4))
    rx = xs + rng.normal(0, 0.1, xs.shape)
    ru = us + rng.normal(0, 0.1, us.shape)
    om = oracle.OracleModel.random_net(list(sizes), "silu", seed, True)
    z = np.concatenate([xs[:, :n, :], us], axis=-1).reshape(-1, 17)
    f, j, h = om.batched_eval(z, order)
    return xs, us, rx, ru, z, f, j, h, om


def test_oracle_binding_matches_linear_residual_naive_identity(oracle_lib):
    """Hover with a zero residual: phi_res vanishes when x_{k+1} is the RK4 step,
    A has the exact RK4 structure (dp/dp = I) and the cost terms follow
    sqp_rti.cpp:143-153 bit-for-bit."""
    p = qp.QuadParams()
    cfg = qp.OcpConfig(horizon=3, dt=0.02, q_diag=np.arange(1, 14.0), r_diag=np.full(4, 0.5))
    x = np.zeros(13)
    x[3] = 1.0
    xs = np.tile(x, (1, 4, 1))
    us = np.full((1, 3, 4), p.hover_thrust_per_rotor())
    rx = xs + 0.25
    ru = us - 0.5
    z = np.concatenate([xs[:, :3], us], axis=-1).reshape(-1, 17)
    out = oracle.build_qp_quad(p.flat(), cfg.flat(), 3, 0, 1, xs, us, rx, ru, z, np.zeros((3, 6)),
                               np.zeros((3, 6, 17)))
    assert np.max(np.abs(out["phi_res"])) < 1e-12
    assert np.array_equal(out["a"][0, :, 0:3, 0:3], np.broadcast_to(np.eye(3), (3, 3, 3)))
    assert np.array_equal(out["q"][0], np.broadcast_to(2.0 * (cfg.q_diag * -0.25), (4, 13)))
    assert np.array_equal(out["r"][0], np.full((3, 4), 2.0 * (0.5 * 0.5)))
    assert np.array_equal(out["du_lb"][0], -us[0])
    assert out["f_evals"] == (12, 12)


def test_oracle_blocks_error_message(oracle_lib):
    xs, us, rx, ru, z, f, j, _, _ = _quad_case(2, 5)
    xs[1, 2, 3] = 3.0  # instance 1, node 2: |q| far from 1 (dynamics.cpp:70-73)
    with pytest.raises(oracle.OracleError, match="instance 1: build qp: node 2: quad dynamics: quaternion norm"):
        oracle.build_qp_quad(qp.QuadParams().flat(), qp.OcpConfig(horizon=5).flat(), 5, 0, 1, xs, us, rx, ru, z, f, j)


def _call_build(params, cfg):
    it, ap, out = _lib.IterateC(), _lib.ApproxC(), _lib.QpBlocksC()
    pc, cc = params.to_c(), cfg.to_c()
    return _lib.lib().rtn_build_qp(None, C.byref(pc), C.byref(cc), 1, C.byref(it), C.byref(ap), C.byref(out), None)


@pytest.mark.parametrize("mutate,msg", [
    (lambda p, c: setattr(p, "mass", 0.0), "quad params: mass, arm_length, torque_coeff, thrust_max must be positive"),
    (lambda p, c: setattr(p, "inertia", (1e-3, -1.0, 1e-3)), "quad params: inertia must be positive"),
    (lambda p, c: setattr(p, "rotor_sign", (1, 1, 1, -1)), "quad params: need two rotors of each spin direction"),
    (lambda p, c: setattr(p, "rotor_sign", (1, 2, -1, -1)), "quad params: rotor_sign entries must be +1 or -1"),
    (lambda p, c: setattr(c, "horizon", 0), "ocp config: horizon must be >= 1"),
    (lambda p, c: setattr(c, "dt", 0.0), "ocp config: dt must be positive"),
    (lambda p, c: c.q_diag.__setitem__(4, -1.0), "ocp config: weights must be nonnegative"),
    (lambda p, c: c.u_min.__setitem__(2, 7.0), "ocp config: u_min must be below u_max"),
    (lambda p, c: setattr(c, "taylor_order", 3), "ocp config: taylor_order must be 1 or 2"),
])
def test_abi_config_errors_match_reference(mutate, msg):
    """sqp_rti.cpp:27-42 / dynamics.cpp:29-40 messages, RTN_ECONFIG, no device needed."""
    p, c = qp.QuadParams(), qp.OcpConfig()
    mutate(p, c)
    st = _call_build(p, c)
    assert st == _lib.RTN_ECONFIG
    with pytest.raises(ConfigError, match=re.escape(msg)):
        raise_for_status(st)


def test_abi_null_context_rejected():
    assert _call_build(qp.QuadParams(), qp.OcpConfig()) == _lib.RTN_ECONFIG
    assert "null argument" in _lib.last_error()
