"""Host mirror of the reference's approximation interface
(/root/reference/proj/include/resmpc/taylor.hpp:13-35, proj/src/taylor.cpp).

`prepare_nodes` is the drop-in boundary: one batched device call for all
nodes (SPEC: "exactly one batched model call per RTI cycle"). `eval_taylor`
and `eval_taylor_jacobian` are the host-side consumers used inside RK4 stages
by the QP builder; they stay on the CPU exactly as in the reference.
"""
from __future__ import annotations

import json
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError
from .neural import EvalCounters, EvalOrder, MlpModel, mlp_batched_eval


@dataclass
class TaylorApprox:
    node: int = 0
    order: int = 1
    z0: np.ndarray = None
    f_bar: np.ndarray = None
    jac: np.ndarray = None                                  # out x in
    hess: list[np.ndarray] = field(default_factory=list)   # per output, order 2 only

    def validate(self) -> None:  # taylor.cpp:9-16
        if self.order not in (1, 2):
            raise ConfigError("taylor: order must be 1 or 2")
        if self.jac.shape != (self.f_bar.size, self.z0.size):
            raise ConfigError("taylor: jacobian shape mismatch")
        if self.order == 2 and len(self.hess) != self.f_bar.size:
            raise ConfigError("taylor: hessian stack missing for order 2")
        if self.order == 1 and len(self.hess) != 0:
            raise ConfigError("taylor: order 1 must not carry hessians")

    def to_json(self) -> str:  # taylor.cpp:18-35
        d = {"node": self.node, "order": self.order, "z0": self.z0.tolist(), "f_bar": self.f_bar.tolist(),
             "jac": self.jac.tolist()}
        if self.hess:
            d["hess"] = [h.tolist() for h in self.hess]
        return json.dumps(d, separators=(",", ":"))


def prepare_nodes(model: MlpModel, node_features, order: int, counters: EvalCounters | None = None,
                  **kw) -> list[TaylorApprox]:
    """taylor.cpp:37-55 — one batched device call for all K nodes."""
    if order not in (1, 2):
        raise ConfigError("prepare nodes: order must be 1 or 2")
    z = np.atleast_2d(np.asarray(node_features, dtype=np.float64))
    batch = mlp_batched_eval(model, z, EvalOrder.HESSIAN if order == 2 else EvalOrder.JACOBIAN, counters, **kw)
    out = []
    for k in range(z.shape[0]):
        a = TaylorApprox(k, order, z[k].copy(), batch.values[k].copy(), batch.jacobians[k].copy(),
                         [batch.hessians[k][o].copy() for o in range(batch.values.shape[1])] if order == 2 else [])
        a.validate()
        out.append(a)
    return out


def eval_taylor(a: TaylorApprox, z) -> np.ndarray:
    """f̄ + J·Δ (+ ½ ΔᵀH_oΔ) — taylor.cpp:57-65."""
    dz = np.asarray(z, dtype=np.float64) - a.z0
    y = a.f_bar + a.jac @ dz
    if a.order == 2:
        y = y + np.array([0.5 * dz @ (h @ dz) for h in a.hess])
    return y


def eval_taylor_jacobian(a: TaylorApprox, z) -> np.ndarray:
    """J (+ H_o·Δ rows) — taylor.cpp:67-74."""
    if a.order == 1:
        return a.jac
    dz = np.asarray(z, dtype=np.float64) - a.z0
    return a.jac + np.stack([h @ dz for h in a.hess])
