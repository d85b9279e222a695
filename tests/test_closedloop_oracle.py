"""CPU tests of the closed-loop trajectory harness (oracle/closedloop_oracle.cpp,
test infrastructure): pinned by the reference's QP tests
(proj/tests/test_qp.cpp:55-221, re-expressed in oracle/test_closedloop.cpp),
and the Python callback route is bit-identical to the in-oracle phase 1."""
import subprocess

import numpy as np

import oracle
from paper_2203_07747_b200 import qp

Q = np.array([10, 10, 10, 1, 1, 1, 1, 1, 1, 1, .1, .1, .1])


def test_reference_qp_and_closed_loop_tests_restated(oracle_lib):
    r = subprocess.run([oracle.os.path.join(oracle.HERE, "build", "test_closedloop")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_callback_phase1_is_bit_identical(oracle_lib):
    p, cfg = qp.QuadParams(), qp.OcpConfig(horizon=20, dt=0.05, q_diag=Q, r_diag=np.full(4, .1))
    om = oracle.OracleModel.random_net([17, 64, 64, 6], "silu", 3, True)
    r0 = oracle.closed_loop(om, p.flat(), cfg.flat(), 20, 1, duration=0.3)
    r1 = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, 1, duration=0.3,
                            prepare=lambda z, o: om.batched_eval(z, o))
    assert not r0["failed"] and len(r0["states"]) == 30 and r0["ok"].all()
    assert np.array_equal(r0["states"], r1["states"]) and np.array_equal(r0["commands"], r1["commands"])
    assert not r1["callback_errors"]


def test_blocks_callback_matches_oracle_buildqp(oracle_lib):
    """Phase 1+2 through the callback route with the oracle's own BuildQp
    reproduces the in-oracle loop bit-for-bit."""
    p, cfg = qp.QuadParams(), qp.OcpConfig(horizon=10, dt=0.05, q_diag=Q, r_diag=np.full(4, .1))
    om = oracle.OracleModel.random_net([17, 32, 6], "tanh", 5, True)

    def blocks(xs, us, rxs, rus):
        z = np.concatenate([xs[:10], us], axis=1)
        f, j, _ = om.batched_eval(z, 1)
        out = oracle.build_qp_quad(p.flat(), cfg.flat(), 10, 0, 1, xs, us, rxs, rus, z, f, j)
        return {k: v[0] for k, v in out.items() if k != "f_evals"}

    r0 = oracle.closed_loop(om, p.flat(), cfg.flat(), 10, 1, duration=0.2)
    r1 = oracle.closed_loop(None, p.flat(), cfg.flat(), 10, 1, duration=0.2, blocks=blocks)
    assert np.array_equal(r0["states"], r1["states"]), np.abs(r0["states"] - r1["states"]).max()
