"""GPU parity of the batched feedback solve (csrc/rtn_qpsolve.cu, SURVEY.md §8f
rank 4) against the oracle's SolveFeedback (oracle/closedloop_oracle.cpp ←
proj/src/sqp_rti.cpp:157-180, proj/src/qp.cpp:33-208), through rtn_solve_feedback.

The QP data come from the oracle's BuildQp on quadrotor iterates (the real
pipeline), fp64 on both sides: steps and recovered states agree to 1e-9 in the
reference metric, statuses match, and the active-set paths (iteration counts,
final working sets) match."""
import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import _lib, qp

pytestmark = pytest.mark.gpu

TOL = 1e-9


def _setup(n_inst, n, seed=3, u_lo=0.0, u_hi=6.0, spread=0.1):
    rng = np.random.default_rng(seed)
    xs = np.empty((n_inst, n + 1, 13))
    xs[..., 0:3] = rng.uniform(-2, 2, (n_inst, n + 1, 3))
    q = rng.uniform(-1, 1, (n_inst, n + 1, 4))
    xs[..., 3:7] = q / np.linalg.norm(q, axis=-1, keepdims=True)
    xs[..., 7:10] = rng.uniform(-1, 1, (n_inst, n + 1, 3))
    xs[..., 10:13] = rng.uniform(-1, 1, (n_inst, n + 1, 3))
    us = rng.uniform(1.0, 3.0, (n_inst, n, 4))
    rx = xs + rng.normal(0, spread, xs.shape)
    ru = us + rng.normal(0, spread, us.shape)
    xm = xs[:, 0, :] + rng.normal(0, spread, (n_inst, 13))
    p = qp.QuadParams()
    cfg = qp.OcpConfig(horizon=n, dt=0.05, q_diag=rng.uniform(0.5, 10, 13), r_diag=rng.uniform(0.05, 1, 4),
                       u_min=np.full(4, u_lo), u_max=np.full(4, u_hi))
    om = oracle.OracleModel.random_net([17, 32, 6], "silu", seed, True)
    z = np.concatenate([xs[:, :n, :], us], axis=-1).reshape(-1, 17)
    f, j, _ = om.batched_eval(z, 1)
    qd = oracle.build_qp_quad(p.flat(), cfg.flat(), n, 0, 1, xs, us, rx, ru, z, f, j)
    qpd = qp.QpData(13, 4, n, *(qd[k] for k in ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb",
                                                  "du_ub")))
    return cfg, qpd, qd, xm, xs, us, om


def _err(a, b):
    a = a.reshape(a.shape[0], -1)
    b = b.reshape(b.shape[0], -1)
    return float(np.max(np.max(np.abs(a - b), axis=1) / (1.0 + np.max(np.abs(b), axis=1))))


def _builder(om):
    return qp.QpBuilder(oracle.to_product_model(om))


@pytest.mark.parametrize("n_inst,n,u_lo,u_hi,status", [(7, 20, 0.0, 6.0, 0), (64, 20, 1.5, 2.2, 0),
                                                        (9, 50, 0.0, 6.0, 0), (9, 50, 1.6, 2.1, 1),
                                                        (5, 60, 0.0, 6.0, 0)])
def test_feedback_matches_oracle(n_inst, n, u_lo, u_hi, status):
    """The fourth case binds so many of the 200 inputs that the primal active-set
    method reaches its 200-pass cap (QpStatus::kMaxIter, qp.cpp:199-207) on both sides:
    the capped iterates agree as well. The factor lives in shared memory as full
    rows (N = 20), as the packed lower triangle (N = 50) and in the global
    workspace (N = 60)."""
    cfg, qpd, qd, xm, xs, us, om = _setup(n_inst, n, seed=n_inst + n, u_lo=u_lo, u_hi=u_hi)
    ref = oracle.solve_feedback(n, qd, xm, xs, us)
    got = _builder(om).solve_feedback(cfg, qpd, xm, xs, us)
    assert np.array_equal(got.status, ref["status"])
    assert (got.status == status).all()
    assert _err(got.dus, ref["dus"]) < TOL and _err(got.dxs, ref["dxs"]) < TOL
    assert _err(got.u_command, ref["u_command"]) < TOL
    assert np.array_equal(got.iterations, ref["iterations"])
    assert np.array_equal(got.active, ref["active"])
    if u_hi - u_lo < 1.0:  # tight bounds: the working sets are not empty
        assert (np.abs(got.active).sum(axis=1) > 0).any()


def test_feedback_warm_start_converges_immediately():
    """test_qp.cpp:195-213: warm-starting from the solution's working set."""
    cfg, qpd, qd, xm, xs, us, om = _setup(16, 20, seed=5, u_lo=1.6, u_hi=2.1)
    b = _builder(om)
    cold = b.solve_feedback(cfg, qpd, xm, xs, us)
    warm = b.solve_feedback(cfg, qpd, xm, xs, us, active=cold.active)
    ref = oracle.solve_feedback(20, qd, xm, xs, us, active=cold.active)
    assert (warm.iterations <= 2).all()
    assert np.array_equal(warm.iterations, ref["iterations"])
    assert _err(warm.dus, cold.dus) < 1e-12


def test_feedback_error_statuses():
    """SolveFeedback throws on a non-finite measured state (sqp_rti.cpp:159-160) and
    SolveBoxQp on crossed bounds (qp.cpp:107-108): per-instance status 2, other
    instances unaffected."""
    cfg, qpd, qd, xm, xs, us, om = _setup(4, 10, seed=9)
    xm = xm.copy()
    xm[1, 5] = np.nan
    lb = qpd.du_lb.copy()
    lb[3, 2, 1] = qpd.du_ub[3, 2, 1] + 1.0
    qpd.du_lb = lb
    qd = dict(qd)
    qd["du_lb"] = lb
    got = _builder(om).solve_feedback(cfg, qpd, xm, xs, us)
    ref = oracle.solve_feedback(10, qd, xm, xs, us)
    assert list(got.status) == [0, 2, 0, 2] == list(ref["status"])
    ok = np.array([0, 2])
    assert _err(got.dus[ok], ref["dus"][ok]) < TOL


def test_feedback_after_device_blocks_end_to_end():
    """Phases 2+3 on the device: rtn_build_qp's blocks feed rtn_solve_feedback;
    the command matches the oracle's BuildQp + SolveFeedback."""
    cfg, qpd, qd, xm, xs, us, om = _setup(12, 20, seed=13, u_lo=1.5, u_hi=2.3)
    b = _builder(om)
    n = 20
    z = np.concatenate([xs[:, :n, :], us], axis=-1).reshape(-1, 17)
    f, j, _ = om.batched_eval(z, 1)
    rng = np.random.default_rng(14)
    rx = xs + rng.normal(0, 0.1, xs.shape)
    ru = us + rng.normal(0, 0.1, us.shape)
    dev_qp = b.build_qp(qp.QuadParams(), cfg, xs, us, rx, ru, {"z0": z, "f_bar": f, "jac": j})
    got = b.solve_feedback(cfg, dev_qp, xm, xs, us)
    ref_qp = oracle.build_qp_quad(qp.QuadParams().flat(), cfg.flat(), n, 0, 1, xs, us, rx, ru, z, f, j)
    ref = oracle.solve_feedback(n, ref_qp, xm, xs, us)
    assert np.array_equal(got.status, ref["status"])
    assert _err(got.u_command, ref["u_command"]) < 1e-9
