"""Closed-loop trajectory parity (north star: "the check covers f, A, B, and the
closed-loop state trajectory over a fixed rollout"). The same RTI rollout of
the quadrotor (oracle/closedloop_oracle.cpp ← proj/src/sqp_rti.cpp, qp.cpp,
simharness.cpp: circle reference, drag + seeded noise, 100 Hz, N = 20) runs with
  - the oracle's fp64 PrepareNodes (the reference path), and
  - the device path through its C-ABI: rtn_prepare (phase 1), or the fused
    rtn_cycle_qp (phases 1+2: approximations + RK4 continuity blocks).
Per-step state error ‖x_dev − x_ref‖∞/(1+‖x_ref‖∞) (proj/tests/oracles.hpp:30-32),
max over the rollout: 1e-3 in TF32/BF16 mode, 1e-5 in 3xTF32 mode."""
import numpy as np
import pytest

import oracle
from paper_2203_07747_b200 import _lib, qp

pytestmark = pytest.mark.gpu

Q = np.array([10, 10, 10, 1, 1, 1, 1, 1, 1, 1, .1, .1, .1])


def _setup(sizes, order, act="silu", seed=3):
    p = qp.QuadParams()
    cfg = qp.OcpConfig(horizon=20, dt=0.05, q_diag=Q, r_diag=np.full(4, .1), taylor_order=order)
    om = oracle.OracleModel.random_net(sizes, act, seed, True)
    return p, cfg, om


def _traj_err(a, b):
    assert a.shape == b.shape
    return float(np.max(np.max(np.abs(a - b), axis=1) / (1.0 + np.max(np.abs(b), axis=1))))


def _device_prepare(om, precision):
    eng = oracle.to_product_model(om).engine(precision=precision, latency_mode=1)

    def prepare(z, order):
        r = eng.prepare(z, order)
        return r.values, r.jacobians, r.hessians
    return prepare


def _device_cycle(om, p, cfg, precision):
    b = qp.QpBuilder(oracle.to_product_model(om), precision=precision, latency_mode=1)

    def blocks(xs, us, rxs, rus):
        d = b.cycle_qp(p, cfg, xs, us, rxs, rus)
        return {n: getattr(d, n)[0] for n in ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub")}
    return blocks


@pytest.mark.parametrize("prec,tol", [("tf32", 1e-3), ("3xtf32", 1e-5), ("bf16x3", 1e-3)])
def test_closed_loop_rollout_matches_oracle_cfg3(prec, tol):
    """cfg3 network (12x512 SiLU), first order, 0.5 s = 50 RTI cycles."""
    p, cfg, om = _setup([17] + [512] * 12 + [6], 1)
    ref = oracle.closed_loop(om, p.flat(), cfg.flat(), 20, 1, duration=0.5)
    assert not ref["failed"] and ref["ok"].all()
    dev = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, 1, duration=0.5,
                             prepare=_device_prepare(om, _lib.PRECISIONS[prec]))
    assert not dev["callback_errors"] and not dev["failed"]
    e_state = _traj_err(dev["states"], ref["states"])
    e_cmd = _traj_err(dev["commands"], ref["commands"])
    assert e_state < tol and e_cmd < 100 * tol, (prec, e_state, e_cmd)
    fused = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, 1, duration=0.5,
                               blocks=_device_cycle(om, p, cfg, _lib.PRECISIONS[prec]))
    assert not fused["callback_errors"] and not fused["failed"]
    assert _traj_err(fused["states"], ref["states"]) < tol


def test_closed_loop_second_order():
    """Order 2 (device Hessians) on a 3x128 SiLU net: the oracle's HessianSingle
    is too slow for 12x512 inside a 50-cycle loop."""
    p, cfg, om = _setup([17, 128, 128, 128, 6], 2)
    ref = oracle.closed_loop(om, p.flat(), cfg.flat(), 20, 2, duration=0.5)
    assert not ref["failed"]
    for prec, tol in (("3xtf32", 1e-5), ("bf16x3", 1e-3)):
        dev = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, 2, duration=0.5,
                                 prepare=_device_prepare(om, _lib.PRECISIONS[prec]))
        assert not dev["callback_errors"]
        assert _traj_err(dev["states"], ref["states"]) < tol, prec
        fused = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, 2, duration=0.5,
                                   blocks=_device_cycle(om, p, cfg, _lib.PRECISIONS[prec]))
        assert not fused["callback_errors"]
        assert _traj_err(fused["states"], ref["states"]) < tol, prec


@pytest.mark.parametrize("prec,tol", [("tf32", 1e-3), ("3xtf32", 1e-5), ("bf16x3", 1e-3)])
def test_closed_loop_conditioned_cfg3(prec, tol):
    """Well-conditioned 12x512 residual (hidden weights x2.5: |J| ~ 0.6, where single-pass
    TF32 misses 1e-3 on f/J themselves). Measured on B200: state error
    TF32 7e-5, 3xTF32 4e-6, bf16x3 2e-6 over 50 cycles (scripts/closedloop_probe2.py)."""
    p, cfg, om = _setup([17] + [512] * 12 + [6], 1)
    for l, (w, b) in enumerate(om.layers()):
        if l < 12:
            om.set_layer(l, w * 2.5, b)
    ref = oracle.closed_loop(om, p.flat(), cfg.flat(), 20, 1, duration=0.5)
    assert not ref["failed"] and ref["ok"].all()
    dev = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, 1, duration=0.5,
                             blocks=_device_cycle(om, p, cfg, _lib.PRECISIONS[prec]))
    assert not dev["callback_errors"] and not dev["failed"]
    assert _traj_err(dev["states"], ref["states"]) < tol, prec
