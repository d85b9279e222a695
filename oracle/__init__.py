"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes binding of oracle/build/liboracle.so: the Eigen-free fp64 CPU
restatement of the reference's hot path (see resmpc_oracle.h). Only tests/,
__graft_entry__.smoke() and bench.py's CPU legs may import this package, and
only as the checker / CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "liboracle.so")
TEST_BIN = os.path.join(HERE, "build", "test_oracle")
TEST_BLOCKS_BIN = os.path.join(HERE, "build", "test_blocks")
ACTS = ("tanh", "relu", "silu")

_lib = None
_dp = C.POINTER(C.c_double)


def build() -> None:
    subprocess.run(["make", "-C", HERE, "-j4", "all"], check=True, stdout=subprocess.DEVNULL)


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        L.oracle_last_error.restype = C.c_char_p
        vp = C.c_void_p
        L.oracle_make_mlp.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_ulonglong, C.POINTER(vp)]
        L.oracle_random_net.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_int, C.c_ulonglong, C.c_int, C.POINTER(vp)]
        L.oracle_load_model.argtypes = [C.c_char_p, C.POINTER(vp)]
        L.oracle_save_model.argtypes = [vp, C.c_char_p]
        L.oracle_free_model.argtypes = [vp]
        L.oracle_free_model.restype = None
        L.oracle_model_info.argtypes = [vp, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.oracle_get_layer.argtypes = [vp, C.c_int, _dp, _dp]
        L.oracle_set_layer.argtypes = [vp, C.c_int, _dp, _dp]
        L.oracle_get_norm.argtypes = [vp, _dp, _dp, _dp, _dp]
        L.oracle_set_norm.argtypes = [vp, _dp, _dp, _dp, _dp]
        L.oracle_batched_eval.argtypes = [vp, _dp, C.c_longlong, C.c_int, C.c_int, _dp, _dp, _dp]
        L.oracle_forward_mode.argtypes = [vp, _dp, C.c_longlong, C.c_int, _dp, _dp, _dp]
        L.oracle_single.argtypes = [vp, _dp, C.c_int, _dp]
        L.oracle_quad_nodes.argtypes = [C.c_ulonglong, C.c_longlong, _dp]
        L.oracle_quad_nodes.restype = None
        L.oracle_random_vector.argtypes = [C.c_ulonglong, C.c_int, C.c_double, C.c_double, _dp]
        L.oracle_random_vector.restype = None
        L.oracle_blocks_last_error.restype = C.c_char_p
        L.oracle_build_qp_quad.argtypes = ([_dp, _dp, C.c_int, C.c_int, C.c_int, C.c_longlong] + [_dp] * 8 +
                                           [_dp] * 9 + [C.POINTER(C.c_ulonglong), C.c_int, _dp])
        L.oracle_quad_dynamics.argtypes = [_dp] * 6
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(_dp) if a is not None else None


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(st):
    if st != 0:
        raise OracleError(st, lib().oracle_last_error().decode())


class OracleModel:
    """Handle on an oracle::MlpModel."""

    def __init__(self, handle):
        self.h = C.c_void_p(handle) if not isinstance(handle, C.c_void_p) else handle

    @classmethod
    def make_mlp(cls, sizes, act="tanh", seed=0):
        h = C.c_void_p()
        s = (C.c_int * len(sizes))(*sizes)
        _check(lib().oracle_make_mlp(s, len(sizes), ACTS.index(act), seed, C.byref(h)))
        return cls(h)

    @classmethod
    def random_net(cls, sizes, act="tanh", rng_seed=0, random_norm=True):
        h = C.c_void_p()
        s = (C.c_int * len(sizes))(*sizes)
        _check(lib().oracle_random_net(s, len(sizes), ACTS.index(act), rng_seed, int(random_norm), C.byref(h)))
        return cls(h)

    @classmethod
    def load(cls, path):
        h = C.c_void_p()
        _check(lib().oracle_load_model(path.encode(), C.byref(h)))
        return cls(h)

    def save(self, path):
        _check(lib().oracle_save_model(self.h, path.encode()))

    def __del__(self):
        try:
            lib().oracle_free_model(self.h)
        except Exception:
            pass

    def info(self):
        n = C.c_int()
        act = C.c_int()
        lib().oracle_model_info(self.h, C.byref(n), None, C.byref(act))
        sizes = (C.c_int * n.value)()
        lib().oracle_model_info(self.h, C.byref(n), sizes, C.byref(act))
        return list(sizes), ACTS[act.value]

    @property
    def sizes(self):
        return self.info()[0]

    def layers(self):
        sizes = self.sizes
        out = []
        for l in range(len(sizes) - 1):
            w = np.empty((sizes[l + 1], sizes[l]))
            b = np.empty(sizes[l + 1])
            _check(lib().oracle_get_layer(self.h, l, _p(w), _p(b)))
            out.append((w, b))
        return out

    def set_layer(self, l, w, b):
        w = np.ascontiguousarray(w, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        _check(lib().oracle_set_layer(self.h, l, _p(w), _p(b)))

    def norm(self):
        s = self.sizes
        v = [np.empty(s[0]), np.empty(s[0]), np.empty(s[-1]), np.empty(s[-1])]
        lib().oracle_get_norm(self.h, *[_p(x) for x in v])
        return v

    def set_norm(self, in_mean, in_scale, out_mean, out_scale):
        v = [np.ascontiguousarray(x, dtype=np.float64) for x in (in_mean, in_scale, out_mean, out_scale)]
        lib().oracle_set_norm(self.h, *[_p(x) for x in v])

    def batched_eval(self, z, order, threads=0):
        """Reverse-mode reference algorithm: returns (f, jac, hess)."""
        z = np.ascontiguousarray(z, dtype=np.float64)
        k = z.shape[0]
        s = self.sizes
        n_in, n_out = s[0], s[-1]
        f = np.empty((k, n_out))
        jac = np.empty((k, n_out, n_in)) if order >= 1 else None
        hess = np.empty((k, n_out, n_in, n_in)) if order >= 2 else None
        _check(lib().oracle_batched_eval(self.h, _p(z), k, order, threads, _p(f), _p(jac), _p(hess)))
        return f, jac, hess

    def forward_mode(self, z, order):
        z = np.ascontiguousarray(z, dtype=np.float64)
        k = z.shape[0]
        s = self.sizes
        n_in, n_out = s[0], s[-1]
        f = np.empty((k, n_out))
        jac = np.empty((k, n_out, n_in))
        hess = np.empty((k, n_out, n_in, n_in)) if order >= 2 else None
        _check(lib().oracle_forward_mode(self.h, _p(z), k, order, _p(f), _p(jac), _p(hess)))
        return f, jac, hess


def quad_nodes(seed, k):
    z = np.empty((k, 17))
    lib().oracle_quad_nodes(seed, k, _p(z))
    return z


def rel_error(a, b) -> float:
    """‖a−b‖∞/(1+‖b‖∞) — proj/tests/oracles.hpp:30-32."""
    a = np.asarray(a)
    b = np.asarray(b)
    return float(np.max(np.abs(a - b)) / (1.0 + np.max(np.abs(b)))) if a.size else 0.0


def max_node_rel_error(a, b) -> float:
    """Per node (axis 0), per block: max over nodes of rel_error."""
    a = np.asarray(a).reshape(a.shape[0], -1)
    b = np.asarray(b).reshape(b.shape[0], -1)
    if a.shape[0] == 0:
        return 0.0
    num = np.max(np.abs(a - b), axis=1)
    den = 1.0 + np.max(np.abs(b), axis=1)
    return float(np.max(num / den))


def to_product_model(om: OracleModel):
    """Copies an oracle model into the product's MlpModel (test helper)."""
    from paper_2203_07747_b200.neural import MlpModel
    sizes, act = om.info()
    layers = om.layers()
    im, isc, outm, outs = om.norm()
    return MlpModel(sizes, [w for w, _ in layers], [b for _, b in layers], act, "full", im, isc, outm, outs, 0)


# ---------------------------------------------------------------------------
# Continuity-block builder oracle (blocks_oracle.h): BuildQp for the quadrotor
# 'full' plant, batched over instances (instance-major rows).
VARIANTS = {"a": (0, 3, 3), "a_u": (1, 7, 3), "full": (2, 17, 6), "ground": (3, 26, 3)}  # code, n_f, n_r


def build_qp_quad(params_flat, cfg_flat, horizon, has_qf, order, xs, us, ref_xs, ref_us, z0, f_bar, jac, hess=None,
                  variant="full", aux=None):
    """Returns dict of QpData arrays + 'f_evals'. Raises OracleError with the
    reference's message ("build qp: node k: ...") on failure. variant: a, a_u,
    full, ground (aux: n_inst x N x 9 height patches)."""
    n = int(horizon)
    code, nf, nr = VARIANTS[variant]
    xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1, n + 1, 13)
    n_inst = xs.shape[0]
    k = n_inst * n
    cast = lambda a, s: np.ascontiguousarray(a, dtype=np.float64).reshape(s)
    ins = [cast(params_flat, (11,)), cast(cfg_flat, (39,))]
    arrs = [xs, cast(us, (n_inst, n, 4)), cast(ref_xs, (n_inst, n + 1, 13)), cast(ref_us, (n_inst, n, 4)),
            cast(z0, (k, nf)), cast(f_bar, (k, nr)), cast(jac, (k, nr, nf)),
            cast(hess, (k, nr, nf, nf)) if order == 2 else None]
    aux_a = cast(aux, (k, 9)) if variant == "ground" else None
    out = {"a": np.empty((n_inst, n, 13, 13)), "b": np.empty((n_inst, n, 13, 4)), "phi_res": np.empty((n_inst, n, 13)),
           "q": np.empty((n_inst, n + 1, 13)), "r": np.empty((n_inst, n, 4)), "hx_diag": np.empty((n_inst, n + 1, 13)),
           "hu_diag": np.empty((n_inst, n, 4)), "du_lb": np.empty((n_inst, n, 4)), "du_ub": np.empty((n_inst, n, 4))}
    fe = (C.c_ulonglong * 2)()
    st = lib().oracle_build_qp_quad(_p(ins[0]), _p(ins[1]), n, int(has_qf), int(order), n_inst,
                                    *[_p(a) for a in arrs], *[_p(out[k_]) for k_ in
                                                              ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag",
                                                               "du_lb", "du_ub")], fe, code, _p(aux_a))
    if st != 0:
        raise OracleError(st, lib().oracle_blocks_last_error().decode())
    out["f_evals"] = (fe[0], fe[1])
    return out


def quad_dynamics(params_flat, x, u):
    """(dx, fx, fu) of the nominal quadrotor (dynamics.cpp:64-86, integrator.cpp:91-123)."""
    dx, fx, fu = np.empty(13), np.empty((13, 13)), np.empty((13, 4))
    st = lib().oracle_quad_dynamics(_p(np.ascontiguousarray(params_flat, dtype=np.float64)),
                                    _p(np.ascontiguousarray(x, dtype=np.float64)),
                                    _p(np.ascontiguousarray(u, dtype=np.float64)), _p(dx), _p(fx), _p(fu))
    if st != 0:
        raise OracleError(st, lib().oracle_blocks_last_error().decode())
    return dx, fx, fu


# ---------------------------------------------------------------------------
# Closed-loop trajectory check (closedloop_oracle.h): one rollout of the
# quadrotor RTI loop; phase 1 (PrepareNodes) and optionally phases 1+2
# (BuildQp blocks) come from Python callables, e.g. the device path.
PREP_CB = C.CFUNCTYPE(C.c_int, _dp, C.c_int, C.c_int, _dp, _dp, _dp, C.c_void_p)
BLOCKS_CB = C.CFUNCTYPE(C.c_int, _dp, _dp, _dp, _dp, C.c_int, *([_dp] * 9), C.c_void_p)


def closed_loop(om, params_flat, cfg_flat, horizon, order, traj=(0, 5.0, 2.0, 20.0, 1.5, 3.0),
                sim=(0.3, 0.3, 0.15, 0.005, 0.02, 1e-3, 100.0), duration=0.5, seed=7, per_step_noise=False,
                prepare=None, blocks=None, has_qf=False):
    """prepare(z K x 17, order) -> (f K x 6, jac K x 6 x 17, hess or None);
    blocks(xs, us, rxs, rus) -> dict of QpData arrays (a, b, phi_res, q, r, hx_diag, hu_diag, du_lb, du_ub).
    Returns dict(states steps x 13, commands steps x 4, ok steps, failed)."""
    L = lib()
    if not hasattr(L, "_cl_bound"):
        L.oracle_closed_loop_last_error.restype = C.c_char_p
        L.oracle_closed_loop.argtypes = [C.c_void_p, _dp, _dp, C.c_int, C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_double,
                                         C.c_ulonglong, PREP_CB, BLOCKS_CB, C.c_void_p, _dp, _dp,
                                         C.POINTER(C.c_int), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L._cl_bound = True
    errors = []

    def _prep(zp, k, ordr, fp, jp, hp, _u):
        try:
            z = np.ctypeslib.as_array(zp, shape=(k, 17)).copy()
            f, j, h = prepare(z, ordr)
            np.ctypeslib.as_array(fp, shape=(k, 6))[:] = f
            np.ctypeslib.as_array(jp, shape=(k, 6, 17))[:] = j
            if ordr == 2:
                np.ctypeslib.as_array(hp, shape=(k, 6, 17, 17))[:] = h
            return 0
        except Exception as e:  # noqa: BLE001 - reported after the rollout
            errors.append(e)
            return 1

    def _blocks(xp, up, rxp, rup, n, *outs_u):
        try:
            outs = outs_u[:9]
            arr = lambda p, s: np.ctypeslib.as_array(p, shape=s)
            res = blocks(arr(xp, (n + 1, 13)).copy(), arr(up, (n, 4)).copy(), arr(rxp, (n + 1, 13)).copy(),
                         arr(rup, (n, 4)).copy())
            shapes = [(n, 13, 13), (n, 13, 4), (n, 13), (n + 1, 13), (n, 4), (n + 1, 13), (n, 4), (n, 4), (n, 4)]
            names = ["a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub"]
            for p, s, nm in zip(outs, shapes, names):
                arr(p, s)[:] = np.reshape(res[nm], s)
            return 0
        except Exception as e:  # noqa: BLE001 - a BuildQp failure: the cycle reuses the last command
            errors.append(e)
            return 1

    pcb = PREP_CB(_prep) if prepare is not None else C.cast(None, PREP_CB)
    bcb = BLOCKS_CB(_blocks) if blocks is not None else C.cast(None, BLOCKS_CB)
    max_steps = int(round(duration * sim[6])) + 2
    states, commands = np.zeros((max_steps, 13)), np.zeros((max_steps, 4))
    ok = np.zeros(max_steps, dtype=np.int32)
    n_steps, failed = C.c_int(), C.c_int()
    arrd = lambda a: np.ascontiguousarray(a, dtype=np.float64)
    st = L.oracle_closed_loop(om.h if om is not None else None, _p(arrd(params_flat)), _p(arrd(cfg_flat)), horizon,
                              int(has_qf), order, _p(arrd(traj)), _p(arrd(sim)), int(per_step_noise), duration, seed,
                              pcb, bcb, None, _p(states), _p(commands), ok.ctypes.data_as(C.POINTER(C.c_int)),
                              max_steps, C.byref(n_steps), C.byref(failed))
    if st != 0:
        raise OracleError(st, L.oracle_closed_loop_last_error().decode())
    n = n_steps.value
    return {"states": states[:n], "commands": commands[:n], "ok": ok[:n], "failed": bool(failed.value),
            "callback_errors": errors}


def solve_feedback(horizon, qpd, x_meas, xs, us, active=None):
    """oracle SolveFeedback per instance (closedloop_oracle.cpp); qpd: dict/obj of QpData arrays."""
    n = int(horizon)
    get = (lambda k: qpd[k]) if isinstance(qpd, dict) else (lambda k: getattr(qpd, k))
    arr = [np.ascontiguousarray(get(k), dtype=np.float64) for k in
           ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub")]
    xs = np.ascontiguousarray(xs, dtype=np.float64).reshape(-1, n + 1, 13)
    n_inst = xs.shape[0]
    us = np.ascontiguousarray(us, dtype=np.float64).reshape(n_inst, n, 4)
    xm = np.ascontiguousarray(x_meas, dtype=np.float64).reshape(n_inst, 13)
    act = (np.zeros((n_inst, 4 * n), dtype=np.int8) if active is None
           else np.ascontiguousarray(active, dtype=np.int8).reshape(n_inst, 4 * n).copy())
    dxs, dus, u = np.empty((n_inst, n + 1, 13)), np.empty((n_inst, n, 4)), np.empty((n_inst, 4))
    st, it = np.empty(n_inst, dtype=np.int32), np.empty(n_inst, dtype=np.int32)
    L = lib()
    if not hasattr(L, "_fb_bound"):
        ip = C.POINTER(C.c_int)
        L.oracle_solve_feedback.argtypes = [C.c_int, C.c_longlong] + [_dp] * 12 + [C.POINTER(C.c_byte), _dp, _dp, _dp,
                                                                                   ip, ip]
        L._fb_bound = True
    rc = L.oracle_solve_feedback(n, n_inst, *[_p(a) for a in arr], _p(xm), _p(xs), _p(us),
                                 act.ctypes.data_as(C.POINTER(C.c_byte)), _p(dxs), _p(dus), _p(u),
                                 st.ctypes.data_as(C.POINTER(C.c_int)), it.ctypes.data_as(C.POINTER(C.c_int)))
    if rc != 0:
        raise OracleError(rc, L.oracle_closed_loop_last_error().decode())
    return {"dxs": dxs, "dus": dus, "u_command": u, "status": st, "iterations": it, "active": act}
