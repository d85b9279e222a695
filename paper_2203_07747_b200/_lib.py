"""ctypes binding of librtn_mpc.so (include/rtn_mpc.h).

There is deliberately no fallback: if the sm_100a library is missing or the
device is not a B200, every compute call raises.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# RTN_LIB overrides the library path (A/B comparisons of builds on one box).
LIB_PATH = os.environ.get("RTN_LIB", os.path.join(_HERE, "librtn_mpc.so"))

RTN_OK, RTN_ECONFIG, RTN_EDOMAIN, RTN_EUNSUPPORTED, RTN_ECUDA, RTN_ENCCL, RTN_ERUNTIME = range(7)
RTN_TF32, RTN_3XTF32, RTN_BF16, RTN_BF16X3 = range(4)  # include/rtn_mpc.h rtn_precision
PRECISIONS = {"tf32": RTN_TF32, "3xtf32": RTN_3XTF32, "bf16x3": RTN_BF16X3, "bf16": RTN_BF16}
# rtn_variant codes and (n_f, n_r) per residual variant (dynamics.hpp:95-131)
VARIANTS = {"full": (0, 17, 6), "a": (1, 3, 3), "a_u": (2, 7, 3), "ground": (3, 26, 3)}

# Every symbol include/rtn_mpc.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "rtn_model_load_rmlp", "rtn_model_from_arrays", "rtn_model_free", "rtn_model_info", "rtn_model_digest",
    "rtn_ctx_create", "rtn_ctx_free", "rtn_prepare", "rtn_prepare_device",
    "rtn_ctx_set_stream", "rtn_ctx_synchronize", "rtn_ctx_counters", "rtn_ctx_nonfinite",
    "rtn_ctx_set_jacobian_mode", "rtn_last_error",
    "rtn_build_qp", "rtn_build_qp_device", "rtn_cycle_qp", "rtn_solve_feedback",
    "rtn_comm_unique_id", "rtn_comm_create", "rtn_comm_free", "rtn_prepare_partitioned",
    "rtn_prepare_partitioned_device", "rtn_comm_bind_root_outputs", "rtn_prepare_partitioned_p2p",
    "rtn_ipc_export", "rtn_ipc_import", "rtn_ipc_release",
)


# Continuity-block builder structs (include/rtn_mpc.h). Pointers are void* so
# the same structs carry host (rtn_build_qp) or device (rtn_build_qp_device) buffers.
class QuadParamsC(C.Structure):
    _fields_ = [("mass", C.c_double), ("inertia", C.c_double * 3), ("arm_length", C.c_double),
                ("torque_coeff", C.c_double), ("thrust_max", C.c_double), ("rotor_sign", C.c_double * 4)]


class OcpConfigC(C.Structure):
    _fields_ = [("horizon", C.c_int), ("dt", C.c_double), ("q_diag", C.c_double * 13), ("r_diag", C.c_double * 4),
                ("has_q_terminal", C.c_int), ("q_terminal", C.c_double * 13), ("u_min", C.c_double * 4),
                ("u_max", C.c_double * 4), ("taylor_order", C.c_int), ("variant", C.c_int)]


class IterateC(C.Structure):
    _fields_ = [("xs", C.c_void_p), ("us", C.c_void_p), ("ref_xs", C.c_void_p), ("ref_us", C.c_void_p),
                ("aux", C.c_void_p)]


class ApproxC(C.Structure):
    _fields_ = [("z0", C.c_void_p), ("f_bar", C.c_void_p), ("jac", C.c_void_p), ("hess", C.c_void_p)]


class QpBlocksC(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub")]


class FeedbackC(C.Structure):
    _fields_ = [("dxs", C.c_void_p), ("dus", C.c_void_p), ("u_command", C.c_void_p), ("status", C.c_void_p),
                ("iterations", C.c_void_p), ("active", C.c_void_p)]

_lib = None

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_vp = C.c_void_p


def lib() -> C.CDLL:
    """Loads the library once; raises loudly when it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2203_07747_b200.build` "
            "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    L.rtn_last_error.restype = C.c_char_p
    L.rtn_model_load_rmlp.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(_vp)]
    L.rtn_model_from_arrays.argtypes = [_ip, C.c_int, C.c_int, C.POINTER(_dp), C.POINTER(_dp),
                                        _dp, _dp, _dp, _dp, C.c_int, C.c_int, C.POINTER(_vp)]
    L.rtn_model_free.argtypes = [_vp]
    L.rtn_model_free.restype = None
    L.rtn_model_info.argtypes = [_vp, _ip, _ip, _ip, _ip, _ip]
    L.rtn_model_digest.argtypes = [_vp, C.c_char_p, _ip]
    L.rtn_ctx_create.argtypes = [_vp, C.c_longlong, C.c_int, C.c_int, C.POINTER(_vp)]
    L.rtn_ctx_free.argtypes = [_vp]
    L.rtn_ctx_free.restype = None
    L.rtn_prepare.argtypes = [_vp, _dp, C.c_longlong, C.c_int, C.c_int, _dp, _dp, _dp]
    L.rtn_prepare_device.argtypes = [_vp, C.c_void_p, C.c_longlong, C.c_int, C.c_void_p, C.c_void_p,
                                     C.c_void_p]
    L.rtn_ctx_set_stream.argtypes = [_vp, _vp]
    L.rtn_ctx_synchronize.argtypes = [_vp]
    L.rtn_ctx_nonfinite.argtypes = [_vp, _ip, C.c_int]
    L.rtn_ctx_counters.argtypes = [_vp, C.POINTER(C.c_ulonglong), C.POINTER(C.c_ulonglong),
                                   C.POINTER(C.c_ulonglong)]
    L.rtn_build_qp.argtypes = [_vp, C.POINTER(QuadParamsC), C.POINTER(OcpConfigC), C.c_longlong,
                               C.POINTER(IterateC), C.POINTER(ApproxC), C.POINTER(QpBlocksC),
                               C.POINTER(C.c_ulonglong)]
    L.rtn_build_qp_device.argtypes = [_vp, C.POINTER(QuadParamsC), C.POINTER(OcpConfigC), C.c_longlong,
                                      C.POINTER(IterateC), C.POINTER(ApproxC), C.POINTER(QpBlocksC)]
    L.rtn_cycle_qp.argtypes = [_vp, C.POINTER(QuadParamsC), C.POINTER(OcpConfigC), C.c_longlong,
                               C.POINTER(IterateC), C.POINTER(QpBlocksC), _vp, _vp, _vp]
    L.rtn_solve_feedback.argtypes = [_vp, C.POINTER(OcpConfigC), C.c_longlong, C.POINTER(QpBlocksC), _vp,
                                     C.POINTER(IterateC), C.POINTER(FeedbackC)]
    L.rtn_comm_unique_id.argtypes = [C.c_char_p]
    L.rtn_comm_create.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, C.POINTER(_vp)]
    L.rtn_comm_free.argtypes = [_vp]
    L.rtn_comm_free.restype = None
    L.rtn_prepare_partitioned.argtypes = [_vp, _vp, _vp, C.c_longlong, C.c_int, C.c_int, C.c_int, _vp, _vp]
    L.rtn_ctx_set_jacobian_mode.argtypes = [_vp, C.c_int]
    L.rtn_comm_bind_root_outputs.argtypes = [_vp, C.c_int, _vp, _vp, C.c_longlong]
    L.rtn_prepare_partitioned_p2p.argtypes = [_vp, _vp, _vp, C.c_longlong, C.c_int]
    L.rtn_ipc_export.argtypes = [_vp, C.c_char_p]
    L.rtn_ipc_import.argtypes = [C.c_char_p, C.c_int, C.POINTER(_vp)]
    L.rtn_ipc_release.argtypes = [_vp]
    L.rtn_prepare_partitioned_device.argtypes = [_vp, _vp, _vp, C.c_longlong, C.c_int, _vp, _vp, C.c_int, _vp, _vp,
                                                 C.c_int]
    L.rtn_make_mlp.argtypes = [_ip, C.c_int, C.c_ulonglong, C.POINTER(_dp), C.POINTER(_dp)]
    L.rtn_synth_quad_nodes.argtypes = [C.c_ulonglong, C.c_longlong, _dp]
    L.rtn_synth_quad_nodes.restype = None
    for name in EXPORTS:
        if name not in ("rtn_last_error", "rtn_model_free", "rtn_ctx_free", "rtn_comm_free"):
            getattr(L, name).restype = C.c_int
    L.rtn_make_mlp.restype = C.c_int
    _lib = L
    return L


def last_error() -> str:
    return lib().rtn_last_error().decode(errors="replace")
