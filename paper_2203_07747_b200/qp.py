"""Host mirror of the reference's QP-block construction for the quadrotor
plant — the step after PrepareNodes.

    QpData resmpc::BuildQp(plant, cfg, iterate, refs, &approxes, nullptr, ...)
        -- /root/reference/proj/include/resmpc/sqp_rti.hpp:56-59
           /root/reference/proj/src/sqp_rti.cpp:59-155

`build_qp` takes prepared approximations (one TaylorApprox per node, or the
flat arrays `prepare_nodes` produces) and runs the RK4 sensitivities of
f_F + embed·Taylor on the device (csrc/rtn_blocks.cu), for every residual
variant (OcpConfig.variant: full, a, a_u, ground — the feature map and its
Jacobian are re-evaluated at each RK4 stage, dynamics.cpp:125-180). `cycle_qp`
fuses phases 1 and 2 of `RtiController::Cycle` (sqp_rti.cpp:219-231): the
MLP's layer 0 gathers z_k = features(x_k, u_k, aux_k) from the iterate →
PrepareNodes → BuildQp in one device pass. Both batch
over independent MPC instances (leading axis). Errors follow the reference:
ConfigError for bad parameters/config (same messages), RuntimeError
"build qp: node k: ..." for a non-finite stage derivative or a quaternion
outside the dynamics' domain. There is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, raise_for_status
from .neural import MlpModel

NX, NU, NF, NR = 13, 4, 17, 6
KGRAVITY = 9.81


@dataclass
class QuadParams:
    """resmpc::QuadParams (proj/include/resmpc/dynamics.hpp:50-62)."""
    mass: float = 0.75
    inertia: tuple = (2.5e-3, 2.5e-3, 4.3e-3)
    arm_length: float = 0.14
    torque_coeff: float = 0.016
    thrust_max: float = 6.0
    rotor_sign: tuple = (1.0, 1.0, -1.0, -1.0)

    def hover_thrust_per_rotor(self) -> float:
        return self.mass * KGRAVITY / 4.0

    def to_c(self) -> _lib.QuadParamsC:
        c = _lib.QuadParamsC()
        c.mass, c.arm_length, c.torque_coeff, c.thrust_max = self.mass, self.arm_length, self.torque_coeff, self.thrust_max
        c.inertia[:] = [float(v) for v in self.inertia]
        c.rotor_sign[:] = [float(v) for v in self.rotor_sign]
        return c

    def flat(self) -> np.ndarray:  # oracle layout
        return np.array([self.mass, *self.inertia, self.arm_length, self.torque_coeff, self.thrust_max,
                         *self.rotor_sign], dtype=np.float64)


@dataclass
class OcpConfig:
    """resmpc::OcpConfig at quadrotor dimensions (sqp_rti.hpp:22-34); rtn mode."""
    horizon: int = 10
    dt: float = 0.1
    q_diag: np.ndarray = field(default_factory=lambda: np.ones(NX))
    r_diag: np.ndarray = field(default_factory=lambda: np.ones(NU))
    q_terminal: np.ndarray | None = None
    u_min: np.ndarray = field(default_factory=lambda: np.zeros(NU))
    u_max: np.ndarray = field(default_factory=lambda: np.full(NU, 6.0))
    taylor_order: int = 1
    variant: str = "full"  # residual variant: full, a, a_u, ground (dynamics.hpp:95-131)

    def dims(self) -> tuple[int, int]:
        """(n_f, n_r) of the variant's network."""
        if self.variant not in _lib.VARIANTS:
            raise ConfigError(f"unknown residual variant '{self.variant}' (expected a, a_u, full, ground)")
        return _lib.VARIANTS[self.variant][1:]

    def terminal_weight(self) -> np.ndarray:
        return self.q_diag if self.q_terminal is None else self.q_terminal

    def to_c(self) -> _lib.OcpConfigC:
        def vec(v, n, what):
            v = np.asarray(v, dtype=np.float64).ravel()
            if v.size != n:
                raise ConfigError(f"ocp config: {what}")
            return [float(x) for x in v]
        c = _lib.OcpConfigC()
        c.horizon, c.dt, c.taylor_order = int(self.horizon), float(self.dt), int(self.taylor_order)
        self.dims()
        c.variant = _lib.VARIANTS[self.variant][0]
        c.q_diag[:] = vec(self.q_diag, NX, "weight dimensions do not match the plant")
        c.r_diag[:] = vec(self.r_diag, NU, "weight dimensions do not match the plant")
        c.has_q_terminal = 0 if self.q_terminal is None else 1
        c.q_terminal[:] = vec(self.terminal_weight(), NX, "terminal weight dimension mismatch")
        c.u_min[:] = vec(self.u_min, NU, "input bound dimensions do not match the plant")
        c.u_max[:] = vec(self.u_max, NU, "input bound dimensions do not match the plant")
        return c

    def flat(self) -> np.ndarray:  # oracle layout: dt, q13, r4, qf13, umin4, umax4
        return np.concatenate([[self.dt], np.ravel(self.q_diag), np.ravel(self.r_diag),
                               np.ravel(self.terminal_weight()), np.ravel(self.u_min),
                               np.ravel(self.u_max)]).astype(np.float64)


@dataclass
class QpData:
    """resmpc::QpData (proj/include/resmpc/qp.hpp:13-28), batched over
    instances: a[i, k] is instance i's 13x13 block of node k."""
    nx: int
    nu: int
    horizon: int
    a: np.ndarray        # n_inst x N x 13 x 13
    b: np.ndarray        # n_inst x N x 13 x 4
    phi_res: np.ndarray  # n_inst x N x 13
    q: np.ndarray        # n_inst x (N+1) x 13
    r: np.ndarray        # n_inst x N x 4
    hx_diag: np.ndarray  # n_inst x (N+1) x 13
    hu_diag: np.ndarray  # n_inst x N x 4
    du_lb: np.ndarray    # n_inst x N x 4
    du_ub: np.ndarray
    f_evals: tuple = (0, 0)  # FevalCounter (values, jacobians)

    def instance(self, i: int) -> "QpData":
        return QpData(self.nx, self.nu, self.horizon, *(getattr(self, n)[i] for n in _QP_FIELDS),
                      f_evals=self.f_evals)


_QP_FIELDS = ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub")


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data


def _batched(a, tail: tuple, what: str) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.ndim == len(tail):
        a = a[None]
    if a.shape[1:] != tail:
        raise ConfigError(f"build qp: {what} has shape {a.shape}, expected (n_inst,) + {tail}")
    return np.ascontiguousarray(a)


def _approx_arrays(approxes, n_inst: int, n: int, order: int, nf: int = NF, nr: int = NR):
    """TaylorApprox list (per node, instance-major) or dict/tuple of flat arrays."""
    k = n_inst * n
    if isinstance(approxes, dict):
        z0, fb, jac = approxes["z0"], approxes["f_bar"], approxes["jac"]
        hess = approxes.get("hess")
    elif isinstance(approxes, (list, tuple)) and approxes and hasattr(approxes[0], "f_bar"):
        if len(approxes) != k:
            raise ConfigError("build qp: need one prepared approximation per shooting node")
        z0 = np.stack([a.z0 for a in approxes])
        fb = np.stack([a.f_bar for a in approxes])
        jac = np.stack([a.jac for a in approxes])
        hess = np.stack([np.stack(a.hess) for a in approxes]) if order == 2 else None
        for a in approxes:
            if a.order != order:
                raise ConfigError("build qp: approximation order does not match taylor_order")
    else:
        raise ConfigError("build qp: approxes must be TaylorApprox objects or a dict of arrays")
    out = [np.ascontiguousarray(np.reshape(z0, (k, nf)), dtype=np.float64),
           np.ascontiguousarray(np.reshape(fb, (k, nr)), dtype=np.float64),
           np.ascontiguousarray(np.reshape(jac, (k, nr, nf)), dtype=np.float64)]
    out.append(np.ascontiguousarray(np.reshape(hess, (k, nr, nf, nf)), dtype=np.float64) if order == 2 else None)
    if order == 2 and hess is None:
        raise ConfigError("build qp: taylor_order 2 needs Hessians")
    return out


class QpBuilder:
    """Owns the device context (one stream + workspace) the way one
    RtiController owns its model handle (sqp_rti.hpp:107)."""

    def __init__(self, model: MlpModel, device: int = 0, precision: int = _lib.RTN_TF32, latency_mode: int = 0):
        self.model = model
        self.engine = model.engine(device, precision, latency_mode)

    def _outputs(self, n_inst: int, n: int):
        outs = {"a": (n, NX, NX), "b": (n, NX, NU), "phi_res": (n, NX), "q": (n + 1, NX), "r": (n, NU),
                "hx_diag": (n + 1, NX), "hu_diag": (n, NU), "du_lb": (n, NU), "du_ub": (n, NU)}
        arrs = {k: np.empty((n_inst,) + s) for k, s in outs.items()}
        c = _lib.QpBlocksC(*[_ptr(arrs[k]) for k in _QP_FIELDS])
        return arrs, c

    def _iterate(self, cfg: OcpConfig, xs, us, ref_xs, ref_us, aux=None):
        n = int(cfg.horizon)
        xs = _batched(xs, (n + 1, NX), "iterate xs")
        us = _batched(us, (n, NU), "iterate us")
        rx = _batched(ref_xs, (n + 1, NX), "reference xs")
        ru = _batched(ref_us, (n, NU), "reference us")
        if not (xs.shape[0] == us.shape[0] == rx.shape[0] == ru.shape[0]):
            raise ConfigError("build qp: iterate and reference window instance counts differ")
        ax = None
        if cfg.variant == "ground":
            if aux is None:
                raise ConfigError("quadrotor plant: ground features need a 9-entry patch aux per node")
            ax = _batched(aux, (n, 9), "ground patches")
        self._keep = (xs, us, rx, ru, ax)
        return xs, us, rx, ru, _lib.IterateC(_ptr(xs), _ptr(us), _ptr(rx), _ptr(ru), _ptr(ax))

    def solve_feedback(self, cfg: OcpConfig, qpd: QpData, x_measured, xs, us, active=None) -> FeedbackResult:
        """SolveFeedback (sqp_rti.cpp:157-180) for every instance on the device:
        condensing + box QP + recovery. `active` (n_inst x 4N) seeds the working set."""
        return _solve_feedback(self.engine, cfg, qpd, x_measured, xs, us, active)

    def build_qp(self, params: QuadParams, cfg: OcpConfig, xs, us, ref_xs, ref_us, approxes, aux=None) -> QpData:
        """BuildQp in rtn mode from prepared approximations (sqp_rti.cpp:59-155).
        aux: per-node 3x3 height patches (row-major, n_inst x N x 9), ground variant only."""
        if cfg.horizon < 1:
            raise ConfigError("ocp config: horizon must be >= 1")
        nf, nr = cfg.dims()
        xs, us, rx, ru, it = self._iterate(cfg, xs, us, ref_xs, ref_us, aux)
        n_inst, n = xs.shape[0], int(cfg.horizon)
        z0, fb, jac, hess = _approx_arrays(approxes, n_inst, n, int(cfg.taylor_order), nf, nr)
        ap = _lib.ApproxC(_ptr(z0), _ptr(fb), _ptr(jac), _ptr(hess))
        arrs, oc = self._outputs(n_inst, n)
        self.engine._ensure(max(n_inst * n, 1), 1)
        fe = (C.c_ulonglong * 2)()
        pc, cc = params.to_c(), cfg.to_c()
        raise_for_status(_lib.lib().rtn_build_qp(self.engine.ctx_ptr, C.byref(pc), C.byref(cc), n_inst, C.byref(it),
                                                 C.byref(ap), C.byref(oc), fe))
        return QpData(NX, NU, n, *(arrs[k] for k in _QP_FIELDS), f_evals=(fe[0], fe[1]))

    def cycle_qp(self, params: QuadParams, cfg: OcpConfig, xs, us, ref_xs, ref_us, return_approx: bool = False,
                 aux=None):
        """Phases 1+2 of RtiController::Cycle on the device: PrepareNodes at
        z_k = features(x_k, u_k, aux_k) (taylor.cpp:37-55) then BuildQp (sqp_rti.cpp:59-155)."""
        if cfg.horizon < 1:
            raise ConfigError("ocp config: horizon must be >= 1")
        nf, nr = cfg.dims()
        xs, us, rx, ru, it = self._iterate(cfg, xs, us, ref_xs, ref_us, aux)
        n_inst, n = xs.shape[0], int(cfg.horizon)
        k = n_inst * n
        order = int(cfg.taylor_order)
        arrs, oc = self._outputs(n_inst, n)
        f = jac = hess = None
        if return_approx:
            f, jac = np.empty((k, nr)), np.empty((k, nr, nf))
            hess = np.empty((k, nr, nf, nf)) if order == 2 else None
        self.engine._ensure(max(k, 1), max(1, min(order, 2)))
        pc, cc = params.to_c(), cfg.to_c()
        raise_for_status(_lib.lib().rtn_cycle_qp(self.engine.ctx_ptr, C.byref(pc), C.byref(cc), n_inst, C.byref(it),
                                                 C.byref(oc), _ptr(f), _ptr(jac), _ptr(hess)))
        qp = QpData(NX, NU, n, *(arrs[k_] for k_ in _QP_FIELDS), f_evals=(4 * k, 4 * k))
        if return_approx:
            return qp, {"f_bar": f, "jac": jac, "hess": hess}
        return qp


@dataclass
class FeedbackResult:
    """resmpc::FeedbackResult (sqp_rti.hpp:61-68), batched: status 0 optimal,
    1 iteration cap, 2 SolveFeedback threw, 3 not positive definite."""
    dxs: np.ndarray        # n_inst x (N+1) x 13
    dus: np.ndarray        # n_inst x N x 4
    u_command: np.ndarray  # n_inst x 4
    status: np.ndarray     # n_inst
    iterations: np.ndarray
    active: np.ndarray     # n_inst x 4N working set (the next call's warm start)


def _solve_feedback(engine, cfg: OcpConfig, qpd: QpData, x_measured, xs, us, active=None) -> FeedbackResult:
    n = int(cfg.horizon)
    xs = _batched(xs, (n + 1, NX), "iterate xs")
    us = _batched(us, (n, NU), "iterate us")
    xm = np.ascontiguousarray(np.reshape(x_measured, (-1, NX)), dtype=np.float64)
    n_inst = xs.shape[0]
    if xm.shape[0] != n_inst:
        raise ConfigError("feedback: one measured state per instance")
    arrs = [np.ascontiguousarray(np.reshape(getattr(qpd, nm), (n_inst, -1)), dtype=np.float64) for nm in _QP_FIELDS]
    qc = _lib.QpBlocksC(*[_ptr(a) for a in arrs])
    dxs, dus, u = np.empty((n_inst, n + 1, NX)), np.empty((n_inst, n, NU)), np.empty((n_inst, NU))
    st, it = np.empty(n_inst, dtype=np.int32), np.empty(n_inst, dtype=np.int32)
    act = (np.zeros((n_inst, n * NU), dtype=np.int8) if active is None
           else np.ascontiguousarray(np.reshape(active, (n_inst, n * NU)), dtype=np.int8).copy())
    out = _lib.FeedbackC(_ptr(dxs), _ptr(dus), _ptr(u), st.ctypes.data, it.ctypes.data, act.ctypes.data)
    itc = _lib.IterateC(_ptr(xs), _ptr(us), None, None, None)
    engine._ensure(1, 1)
    cc = cfg.to_c()
    raise_for_status(_lib.lib().rtn_solve_feedback(engine.ctx_ptr, C.byref(cc), n_inst, C.byref(qc), _ptr(xm),
                                                   C.byref(itc), C.byref(out)))
    return FeedbackResult(dxs, dus, u, st, it, act)


def build_qp(model: MlpModel, params: QuadParams, cfg: OcpConfig, xs, us, ref_xs, ref_us, approxes,
             aux=None, **kw) -> QpData:
    return QpBuilder(model, **kw).build_qp(params, cfg, xs, us, ref_xs, ref_us, approxes, aux=aux)


def cycle_qp(model: MlpModel, params: QuadParams, cfg: OcpConfig, xs, us, ref_xs, ref_us, aux=None, **kw):
    ret = kw.pop("return_approx", False)
    return QpBuilder(model, **kw).cycle_qp(params, cfg, xs, us, ref_xs, ref_us, return_approx=ret, aux=aux)
