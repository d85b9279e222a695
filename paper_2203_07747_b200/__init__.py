"""B200-native per-node MLP linearisation for Real-time Neural MPC (arXiv 2203.07747).

The product is librtn_mpc.so (sm_100a kernels behind the C-ABI in
include/rtn_mpc.h); this package is the host-side mirror of the reference's
`resmpc::PrepareNodes` / `resmpc::MlpBatchedEval` interface on top of it, plus
the step after it (`resmpc::BuildQp`'s RK4 continuity blocks, qp.py).
"""
from .errors import ConfigError, DeviceError, InputDomainError, UnsupportedError
from .neural import (BatchEval, Engine, EvalCounters, EvalOrder, MlpModel, flops_per_node, load_model, make_mlp,
                     make_zero_network,
                     mlp_batched_eval, mlp_forward, mlp_hessian, mlp_jacobian, parse_arch, save_model,
                     synth_quad_nodes)
from .qp import OcpConfig, QpBuilder, QpData, QuadParams, build_qp, cycle_qp
from .taylor import TaylorApprox, eval_taylor, eval_taylor_jacobian, prepare_nodes

__all__ = [
    "BatchEval", "ConfigError", "DeviceError", "Engine", "EvalCounters", "EvalOrder", "InputDomainError",
    "MlpModel", "TaylorApprox", "UnsupportedError", "eval_taylor", "eval_taylor_jacobian", "flops_per_node",
    "load_model", "make_mlp", "make_zero_network", "mlp_batched_eval", "mlp_forward", "mlp_hessian", "mlp_jacobian", "parse_arch",
    "prepare_nodes", "save_model", "synth_quad_nodes",
    "OcpConfig", "QpBuilder", "QpData", "QuadParams", "build_qp", "cycle_qp",
]
