"""GPU parity of the continuity-block builder (csrc/rtn_blocks.cu) against the
oracle's BuildQp restatement (oracle/blocks_oracle.cpp ← proj/src/sqp_rti.cpp:59-155,
proj/src/integrator.cpp:41-123), through the C-ABI (rtn_build_qp / rtn_cycle_qp).

The block builder is fp64 on both sides, so with identical approximations
the tolerance is 1e-12 in the reference's metric ‖a−b‖∞/(1+‖b‖∞)
(proj/tests/oracles.hpp:30-32), per block, max over nodes."""
import re

import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import ConfigError, _lib, qp
from paper_2203_07747_b200.errors import UnsupportedError

pytestmark = pytest.mark.gpu

FIELDS = ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub")
TOL = 1e-12


def _case(n_inst, n, seed=3, order=1, sizes=(17, 32, 32, 6), act="silu", qn_noise=0.0):
    rng = np.random.default_rng(seed)
    xs = np.empty((n_inst, n + 1, 13))
    xs[..., 0:3] = rng.uniform(-2, 2, (n_inst, n + 1, 3))
    q = rng.uniform(-1, 1, (n_inst, n + 1, 4))
    xs[..., 3:7] = q / np.linalg.norm(q, axis=-1, keepdims=True) * (1.0 + qn_noise)
    xs[..., 7:10] = rng.uniform(-4, 4, (n_inst, n + 1, 3))
    xs[..., 10:13] = rng.uniform(-3, 3, (n_inst, n + 1, 3))
    us = rng.uniform(0.5, 5.0, (n_inst, n, 4))
    rx = xs + rng.normal(0, 0.1, xs.shape)
    ru = us + rng.normal(0, 0.1, us.shape)
    om = oracle.OracleModel.random_net(list(sizes), act, seed, True)
    z = np.concatenate([xs[:, :n, :], us], axis=-1).reshape(-1, 17)
    f, j, h = om.batched_eval(z, order)
    return xs, us, rx, ru, z, f, j, h, om


def _cfg(n, order=1, dt=0.05, qf=False):
    rng = np.random.default_rng(n)
    return qp.OcpConfig(horizon=n, dt=dt, q_diag=rng.uniform(0, 10, 13), r_diag=rng.uniform(0, 1, 4),
                        q_terminal=rng.uniform(0, 20, 13) if qf else None, u_min=np.zeros(4),
                        u_max=np.full(4, 6.0), taylor_order=order)


def _block_err(got, ref):
    """max over blocks of ‖a−b‖∞/(1+‖b‖∞)."""
    g = got.reshape(-1, *got.shape[2:]) if got.ndim > 2 else got
    r = ref.reshape(-1, *ref.shape[2:]) if ref.ndim > 2 else ref
    ax = tuple(range(1, g.ndim))
    return float(np.max(np.max(np.abs(g - r), axis=ax) / (1.0 + np.max(np.abs(r), axis=ax))))


def _oracle_qp(p, cfg, xs, us, rx, ru, z, f, j, h):
    return oracle.build_qp_quad(p.flat(), cfg.flat(), cfg.horizon, cfg.q_terminal is not None, cfg.taylor_order,
                                xs, us, rx, ru, z, f, j, h)


def _model(om):
    return oracle.to_product_model(om)


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("n_inst,n", [(1, 20), (7, 13), (64, 50)])
def test_build_qp_matches_oracle(order, n_inst, n):
    xs, us, rx, ru, z, f, j, h, om = _case(n_inst, n, seed=n_inst + n, order=order)
    p, cfg = qp.QuadParams(), _cfg(n, order, qf=n_inst == 7)
    ref = _oracle_qp(p, cfg, xs, us, rx, ru, z, f, j, h)
    ap = {"z0": z, "f_bar": f, "jac": j, "hess": h if order == 2 else None}
    got = qp.QpBuilder(_model(om)).build_qp(p, cfg, xs, us, rx, ru, ap)
    for name in FIELDS:
        e = _block_err(getattr(got, name), ref[name])
        assert e < TOL, (name, e)
    # bitwise where the reference arithmetic has no rounding choices (sqp_rti.cpp:143-153)
    for name in ("q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub"):
        assert np.array_equal(getattr(got, name), ref[name]), name
    assert got.f_evals == ref["f_evals"] == (4 * n_inst * n, 4 * n_inst * n)


def test_build_qp_accepts_taylor_approx_objects():
    from paper_2203_07747_b200 import TaylorApprox
    xs, us, rx, ru, z, f, j, h, om = _case(1, 6, order=2)
    aps = [TaylorApprox(k, 2, z[k], f[k], j[k], [h[k, o] for o in range(6)]) for k in range(6)]
    p, cfg = qp.QuadParams(), _cfg(6, 2)
    got = qp.build_qp(_model(om), p, cfg, xs[0], us[0], rx[0], ru[0], aps)
    ref = _oracle_qp(p, cfg, xs, us, rx, ru, z, f, j, h)
    assert _block_err(got.a, ref["a"]) < TOL and _block_err(got.b, ref["b"]) < TOL


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("latency", [0, 1])
def test_cycle_qp_fused_matches_oracle(order, latency):
    """Phases 1+2 fused on the device: the blocks equal the oracle's BuildQp on
    the device's own approximations (fp64 parity), and those approximations
    equal the oracle's PrepareNodes within the MLP path's tolerance."""
    n_inst, n = 3, 20
    xs, us, rx, ru, z, f, j, h, om = _case(n_inst, n, seed=11, order=order, sizes=(17, 64, 64, 6))
    p, cfg = qp.QuadParams(), _cfg(n, order)
    b = qp.QpBuilder(_model(om), precision=_lib.RTN_3XTF32, latency_mode=latency)
    for _ in range(3 if latency else 1):  # graph capture, then replays
        got, ap = b.cycle_qp(p, cfg, xs, us, rx, ru, return_approx=True)
        ref = _oracle_qp(p, cfg, xs, us, rx, ru, z, ap["f_bar"], ap["jac"], ap["hess"])
        for name in FIELDS:
            assert _block_err(getattr(got, name), ref[name]) < TOL, name
        assert oracle.max_node_rel_error(ap["f_bar"], f) < 1e-5
        assert oracle.max_node_rel_error(ap["jac"], j) < 1e-5
        if order == 2:
            assert oracle.max_node_rel_error(ap["hess"], h) < 1e-4
    calls, points, launches = b.engine.counters()
    assert points == calls * n_inst * n  # one batched model call of K points per cycle
    assert launches == 2 * calls  # MLP (gathering [x;u] itself) + blocks, per cycle


def test_cycle_qp_blocks_vs_oracle_end_to_end():
    """Whole-path check against the fp64 oracle (oracle PrepareNodes → oracle
    BuildQp) at the MLP path's tolerance (3xTF32)."""
    xs, us, rx, ru, z, f, j, h, om = _case(4, 10, seed=5, sizes=(17, 128, 128, 128, 6))
    p, cfg = qp.QuadParams(), _cfg(10, 1)
    got = qp.cycle_qp(_model(om), p, cfg, xs, us, rx, ru, precision=_lib.RTN_3XTF32)
    ref = _oracle_qp(p, cfg, xs, us, rx, ru, z, f, j, h)
    for name in FIELDS:
        assert _block_err(getattr(got, name), ref[name]) < 1e-5, name


def test_errors_match_reference_messages():
    xs, us, rx, ru, z, f, j, h, om = _case(3, 8)
    p, cfg = qp.QuadParams(), _cfg(8)
    b = qp.QpBuilder(_model(om))
    ap = {"z0": z, "f_bar": f, "jac": j}
    bad = xs.copy()
    bad[2, 5, 3] = 3.0  # quaternion far from unit at instance 2, node 5
    bad[2, 7, 4] = 9.0  # a later node fails too; the lowest one is reported
    with pytest.raises(RuntimeError, match=re.escape(
            "instance 2: build qp: node 5: quad dynamics: quaternion norm too far from unit")):
        b.build_qp(p, cfg, bad, us, rx, ru, ap)
    f2 = f.copy()
    f2[9, 2] = np.inf  # instance 1, node 1: non-finite residual at stage 1
    with pytest.raises(RuntimeError, match=re.escape("instance 1: build qp: node 1: rk4: non-finite derivative at stage 1")):
        b.build_qp(p, cfg, xs, us, rx, ru, {"z0": z, "f_bar": f2, "jac": j})
    # single instance: exactly the reference's message (sqp_rti.cpp:134-138)
    with pytest.raises(RuntimeError, match=r"^build qp: node 5: quad dynamics"):
        b.build_qp(p, cfg, bad[2:3], us[2:3], rx[2:3], ru[2:3], {"z0": z[16:24], "f_bar": f[16:24], "jac": j[16:24]})
    # the builder still works after an error
    ref = _oracle_qp(p, cfg, xs, us, rx, ru, z, f, j, h)
    assert _block_err(b.build_qp(p, cfg, xs, us, rx, ru, ap).a, ref["a"]) < TOL
    cfg_bad = _cfg(8)
    cfg_bad.u_min[1] = 10.0
    with pytest.raises(ConfigError, match="u_min must be below u_max"):
        b.build_qp(p, cfg_bad, xs, us, rx, ru, ap)


def test_cycle_rejects_model_variant_mismatch():
    om = oracle.OracleModel.random_net([6, 16, 4], "tanh", 1, True)
    xs, us, rx, ru, *_ = _case(1, 4)
    with pytest.raises(ConfigError, match="needs 17 -> 6"):
        qp.cycle_qp(_model(om), qp.QuadParams(), _cfg(4), xs, us, rx, ru)
    om = oracle.OracleModel.random_net([17, 16, 6], "relu", 1, True)
    with pytest.raises(UnsupportedError):
        qp.cycle_qp(_model(om), qp.QuadParams(), _cfg(4, 2), xs, us, rx, ru)


def test_stage_quaternion_drift_inside_domain():
    """Interior RK4 stages may drift ‖q‖ (dynamics.cpp:67-69); |‖q‖−1| ≤ 0.25 passes."""
    xs, us, rx, ru, z, f, j, h, om = _case(2, 6, qn_noise=0.1)
    p, cfg = qp.QuadParams(), _cfg(6)
    z = np.concatenate([xs[:, :6, :], us], axis=-1).reshape(-1, 17)
    f, j, _ = om.batched_eval(z, 1)
    got = qp.QpBuilder(_model(om)).build_qp(p, cfg, xs, us, rx, ru, {"z0": z, "f_bar": f, "jac": j})
    ref = _oracle_qp(p, cfg, xs, us, rx, ru, z, f, j, None)
    assert _block_err(got.a, ref["a"]) < TOL and _block_err(got.phi_res, ref["phi_res"]) < TOL


def test_large_batch_sampled_parity():
    """4096 instances x N=20 on the device; the oracle checks a sample of instances."""
    n_inst, n = 4096, 20
    xs, us, rx, ru, z, f, j, h, om = _case(n_inst, n, seed=7)
    p, cfg = qp.QuadParams(), _cfg(n)
    got = qp.QpBuilder(_model(om)).build_qp(p, cfg, xs, us, rx, ru, {"z0": z, "f_bar": f, "jac": j})
    idx = np.array([0, 1, 977, 2048, 4095])
    rows = (idx[:, None] * n + np.arange(n)).ravel()
    ref = _oracle_qp(p, cfg, xs[idx], us[idx], rx[idx], ru[idx], z[rows], f[rows], j[rows], None)
    for name in FIELDS:
        assert _block_err(getattr(got, name)[idx], ref[name]) < TOL, name


def test_empty_batch():
    xs, us, rx, ru, z, f, j, h, om = _case(1, 3)
    got = qp.QpBuilder(_model(om)).build_qp(qp.QuadParams(), _cfg(3), xs[:0], us[:0], rx[:0], ru[:0],
                                             {"z0": z[:0], "f_bar": f[:0], "jac": j[:0]})
    assert got.a.shape == (0, 3, 13, 13)


def test_latency_mode_errors_and_recovery():
    """Latency mode (graph + zero-copy staging, per-node status bytes) reports
    the reference's message for the lowest failing node and recovers."""
    xs, us, rx, ru, z, f, j, h, om = _case(1, 20, seed=21)
    p, cfg = qp.QuadParams(), _cfg(20)
    b = qp.QpBuilder(_model(om), precision=_lib.RTN_BF16X3, latency_mode=1)
    good = b.cycle_qp(p, cfg, xs, us, rx, ru)
    bad = xs.copy()
    bad[0, 11, 5] = 4.0
    bad[0, 14, 3] = np.nan  # non-finite later; node 11's domain error is the one reported
    for _ in range(2):  # first call runs outside the graph, the second replays it
        with pytest.raises(RuntimeError, match=re.escape("build qp: node 11: quad dynamics: quaternion norm too far")):
            b.cycle_qp(p, cfg, bad, us, rx, ru)
    again = b.cycle_qp(p, cfg, xs, us, rx, ru)
    for name in FIELDS:
        assert np.array_equal(getattr(again, name), getattr(good, name)), name
    ap = {"z0": z, "f_bar": f, "jac": j}
    f2 = f.copy()
    f2[3, 0] = np.nan
    with pytest.raises(RuntimeError, match=re.escape("build qp: node 3: rk4: non-finite derivative at stage 1")):
        b.build_qp(p, cfg, xs, us, rx, ru, {"z0": z, "f_bar": f2, "jac": j})
    ref = _oracle_qp(p, cfg, xs, us, rx, ru, z, f, j, None)
    got = b.build_qp(p, cfg, xs, us, rx, ru, ap)
    assert _block_err(got.a, ref["a"]) < TOL


# --- residual variants: features + chain rule on the device ---
VARS = {"a": (3, 3), "a_u": (7, 3), "full": (17, 6), "ground": (26, 3)}


def _variant_case(var, n_inst, n, order, seed=17, hidden=(32, 32)):
    xs, us, rx, ru, *_ = _case(n_inst, n, seed=seed)
    nf, nr = VARS[var]
    rng = np.random.default_rng(seed + 1)
    aux = rng.uniform(-0.3, 0.4, (n_inst, n, 9)) if var == "ground" else None
    x, u = xs[:, :n, :], us
    if var == "full":
        z = np.concatenate([x, u], axis=-1)
    elif var == "ground":
        z = np.concatenate([x, u, x[..., 2:3] - aux], axis=-1)
    else:
        q, v = x[..., 3:7], x[..., 7:10]
        w_, x_, y_, z_ = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
        R = np.stack([np.stack([1 - 2 * (y_ * y_ + z_ * z_), 2 * (x_ * y_ - w_ * z_), 2 * (x_ * z_ + w_ * y_)], -1),
                      np.stack([2 * (x_ * y_ + w_ * z_), 1 - 2 * (x_ * x_ + z_ * z_), 2 * (y_ * z_ - w_ * x_)], -1),
                      np.stack([2 * (x_ * z_ - w_ * y_), 2 * (y_ * z_ + w_ * x_), 1 - 2 * (x_ * x_ + y_ * y_)], -1)], -2)
        vb = np.einsum("...ij,...i->...j", R, v)  # Rᵀ v
        z = vb if var == "a" else np.concatenate([vb, u], axis=-1)
    z = z.reshape(-1, nf)
    om = oracle.OracleModel.random_net([nf, *hidden, nr], "silu", seed, True)
    f, j, h = om.batched_eval(z, order)
    return xs, us, rx, ru, z, f, j, h, om, aux


@pytest.mark.parametrize("order", [1, 2])
@pytest.mark.parametrize("var", ["a", "a_u", "full", "ground"])
def test_build_qp_variants_match_oracle(var, order):
    """BuildQp for every residual variant: stage features + jz chain rule
    (dynamics.cpp:125-180, sqp_rti.cpp:96-111) at fp64 parity."""
    n_inst, n = 5, 12
    xs, us, rx, ru, z, f, j, h, om, aux = _variant_case(var, n_inst, n, order)
    p, cfg = qp.QuadParams(), _cfg(n, order)
    cfg.variant = var
    ref = oracle.build_qp_quad(p.flat(), cfg.flat(), n, 0, order, xs, us, rx, ru, z, f, j, h if order == 2 else None,
                               variant=var, aux=aux)
    b = qp.QpBuilder(_model(oracle.OracleModel.random_net([17, 8, 6], "tanh", 1, True)))  # context owner only
    got = b.build_qp(p, cfg, xs, us, rx, ru, {"z0": z, "f_bar": f, "jac": j, "hess": h if order == 2 else None}, aux=aux)
    for name in FIELDS:
        assert _block_err(getattr(got, name), ref[name]) < TOL, (var, order, name)


@pytest.mark.parametrize("var", ["a", "a_u", "ground"])
def test_cycle_qp_variants_fused(var):
    """The fused cycle for every variant: the MLP's layer 0 gathers the variant's
    features from the iterate; blocks match the oracle on the device's own
    approximations (fp64), and those match the oracle PrepareNodes (3xTF32)."""
    n_inst, n = 3, 20
    xs, us, rx, ru, z, f, j, h, om, aux = _variant_case(var, n_inst, n, 1, hidden=(64, 64))
    p, cfg = qp.QuadParams(), _cfg(n, 1)
    cfg.variant = var
    for latency in (0, 1):
        b = qp.QpBuilder(_model(om), precision=_lib.RTN_3XTF32, latency_mode=latency)
        got, ap = b.cycle_qp(p, cfg, xs, us, rx, ru, return_approx=True, aux=aux)
        assert oracle.max_node_rel_error(ap["f_bar"], f) < 1e-5 and oracle.max_node_rel_error(ap["jac"], j) < 1e-5
        ref = oracle.build_qp_quad(p.flat(), cfg.flat(), n, 0, 1, xs, us, rx, ru, z, ap["f_bar"], ap["jac"],
                                   variant=var, aux=aux)
        for name in FIELDS:
            assert _block_err(getattr(got, name), ref[name]) < TOL, (var, latency, name)


def test_variant_model_mismatch_rejected():
    om = oracle.OracleModel.random_net([17, 16, 6], "tanh", 1, True)
    xs, us, rx, ru, *_ = _case(1, 4)
    cfg = _cfg(4)
    cfg.variant = "a"
    with pytest.raises(ConfigError, match="residual wiring"):
        qp.cycle_qp(_model(om), qp.QuadParams(), cfg, xs, us, rx, ru)
    cfg.variant = "ground"
    om3 = oracle.OracleModel.random_net([26, 16, 3], "tanh", 1, True)
    with pytest.raises(ConfigError, match="patch aux"):
        qp.cycle_qp(_model(om3), qp.QuadParams(), cfg, xs, us, rx, ru)
