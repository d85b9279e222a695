"""Host-side mirror of the reference's model interface, backed by the sm_100a
C-ABI (include/rtn_mpc.h).

Names, argument meaning and error behaviour follow
/root/reference/proj/include/resmpc/neural.hpp and proj/src/neural.cpp:
  MlpModel (hpp:19-34), EvalCounters (hpp:38-44), EvalOrder/BatchEval
  (hpp:57-63), MlpForward/MlpJacobian/MlpHessian (hpp:46-55),
  MlpBatchedEval (hpp:65-69), MakeMlp (hpp:105-106), SaveModel/LoadModel
  (hpp:116-117), ParseArch (hpp:120).
Every evaluation goes through the device kernels; nothing here computes the
network on the CPU.
"""
from __future__ import annotations

import ctypes as C
import enum
import json
import math
import os
import struct
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ConfigError, InputDomainError, UnsupportedError, raise_for_status

ACTIVATIONS = ("tanh", "relu", "silu")


class EvalOrder(enum.IntEnum):
    VALUE = 0
    JACOBIAN = 1
    HESSIAN = 2


@dataclass
class EvalCounters:
    value_evals: int = 0
    jacobian_evals: int = 0
    hessian_evals: int = 0
    batched_calls: int = 0
    batched_points: int = 0


@dataclass
class BatchEval:
    values: np.ndarray                    # K x out
    jacobians: np.ndarray | None = None   # K x out x in
    hessians: np.ndarray | None = None    # K x out x in x in


@dataclass(eq=False)
class MlpModel:
    """Dense MLP y = out_scale ⊙ net((z − in_mean) ⊘ in_scale) + out_mean.

    Immutable after the first evaluation (neural.hpp:17-18): the device copy
    is packed once and cached; call `invalidate()` after editing weights.
    """
    layer_sizes: list[int]
    weights: list[np.ndarray]   # weights[l]: sizes[l+1] x sizes[l]
    biases: list[np.ndarray]
    activation: str = "tanh"
    input_variant: str = "full"
    in_mean: np.ndarray = None
    in_scale: np.ndarray = None
    out_mean: np.ndarray = None
    out_scale: np.ndarray = None
    seed: int = 0
    _engines: dict = field(default_factory=dict, repr=False)

    def input_dim(self) -> int:
        return self.layer_sizes[0]

    def output_dim(self) -> int:
        return self.layer_sizes[-1]

    def hidden_layers(self) -> int:
        return len(self.layer_sizes) - 2

    def parameter_count(self) -> int:  # neural.cpp:270-275
        return sum(self.layer_sizes[l + 1] * (self.layer_sizes[l] + 1) for l in range(len(self.layer_sizes) - 1))

    def arch_name(self) -> str:  # neural.cpp:277-281
        return f"N-{self.hidden_layers()}-{self.layer_sizes[1] if self.hidden_layers() > 0 else 0}"

    def validate(self) -> None:  # neural.cpp:283-298
        s = self.layer_sizes
        if len(s) < 2:
            raise ConfigError("mlp: need at least input and output layers")
        if len(self.weights) != len(s) - 1 or len(self.biases) != len(self.weights):
            raise ConfigError("mlp: weight/bias count does not match layer sizes")
        for l, (w, b) in enumerate(zip(self.weights, self.biases)):
            if np.shape(w) != (s[l + 1], s[l]):
                raise ConfigError(f"mlp: layer {l} has incompatible shape")
            if np.shape(b) != (s[l + 1],):
                raise ConfigError(f"mlp: bias {l} has incompatible shape")
        for v, n in ((self.in_mean, s[0]), (self.in_scale, s[0]), (self.out_mean, s[-1]), (self.out_scale, s[-1])):
            if v is None or np.shape(v) != (n,):
                raise ConfigError("mlp: normalization vectors do not match layer sizes")
        if not (np.min(self.in_scale) > 0.0) or not (np.min(self.out_scale) > 0.0):
            raise ConfigError("mlp: normalization scales must be strictly positive")
        if self.activation not in ACTIVATIONS:
            raise ConfigError(f"mlp: unknown activation {self.activation!r}")

    def invalidate(self) -> None:
        for eng in self._engines.values():
            eng.close()
        self._engines.clear()

    def engine(self, device: int = 0, precision: int = _lib.RTN_TF32, latency_mode: int = 0,
               jacobian_mode: int = 0) -> "Engine":
        key = (device, precision, latency_mode, jacobian_mode)
        eng = self._engines.get(key)
        if eng is None:
            eng = Engine(self, device, precision, latency_mode=latency_mode, jacobian_mode=jacobian_mode)
            self._engines[key] = eng
        return eng


def _arr(a) -> C.POINTER(C.c_double):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class Engine:
    """One packed device model plus one context (stream + workspace)."""

    def __init__(self, model: MlpModel, device: int = 0, precision: int = _lib.RTN_TF32,
                 max_rows: int = 1024, latency_mode: int = 0, jacobian_mode: int = 0):
        model.validate()
        L = _lib.lib()
        self.model_ptr = C.c_void_p()
        self.ctx_ptr = C.c_void_p()
        sizes = np.ascontiguousarray(model.layer_sizes, dtype=np.int32)
        ws = [np.ascontiguousarray(w, dtype=np.float64) for w in model.weights]
        bs = [np.ascontiguousarray(b, dtype=np.float64) for b in model.biases]
        wp = (C.POINTER(C.c_double) * len(ws))(*[_arr(w) for w in ws])
        bp = (C.POINTER(C.c_double) * len(bs))(*[_arr(b) for b in bs])
        norm = [np.ascontiguousarray(v, dtype=np.float64)
                for v in (model.in_mean, model.in_scale, model.out_mean, model.out_scale)]
        st = L.rtn_model_from_arrays(sizes.ctypes.data_as(C.POINTER(C.c_int)), len(sizes),
                                     ACTIVATIONS.index(model.activation), wp, bp, *[_arr(v) for v in norm],
                                     device, precision, C.byref(self.model_ptr))
        raise_for_status(st)
        self.n_in, self.n_out = model.input_dim(), model.output_dim()
        self.act = model.activation
        self.max_rows = 0
        self.max_order = 1 if model.activation == "relu" else 1
        self.latency_mode = latency_mode
        self.jacobian_mode = jacobian_mode
        self._ensure(max_rows, 1)

    def _ensure(self, rows: int, order: int) -> None:
        if rows <= self.max_rows and order <= self.max_order and self.ctx_ptr:
            return
        L = _lib.lib()
        if self.ctx_ptr:
            L.rtn_ctx_free(self.ctx_ptr)
            self.ctx_ptr = C.c_void_p()
        self.max_rows = max(rows, self.max_rows, 1)
        self.max_order = max(order, self.max_order)
        raise_for_status(L.rtn_ctx_create(self.model_ptr, self.max_rows, self.max_order, self.latency_mode,
                                          C.byref(self.ctx_ptr)))
        if self.jacobian_mode:
            raise_for_status(L.rtn_ctx_set_jacobian_mode(self.ctx_ptr, self.jacobian_mode))

    def set_jacobian_mode(self, mode: int) -> None:
        """0 = forward mode (default), 1 = reverse mode (rtn_ctx_set_jacobian_mode:
        TF32 models of padded width 512 with n_in <= 24)."""
        raise_for_status(_lib.lib().rtn_ctx_set_jacobian_mode(self.ctx_ptr, mode))
        self.jacobian_mode = mode

    def prepare(self, z: np.ndarray, order: int) -> BatchEval:
        z = np.ascontiguousarray(z, dtype=np.float64)
        if z.ndim != 2:
            raise InputDomainError("mlp eval: expected a K x in matrix of feature rows")
        k, cols = z.shape
        if cols != self.n_in:
            raise InputDomainError(f"mlp eval: feature dim {cols} does not match model input {self.n_in}")
        if order == 2 and self.act == "relu":
            raise UnsupportedError("mlp hessian: only tanh/silu networks are twice differentiable here")
        self._ensure(k, order)
        f = np.empty((k, self.n_out))
        jac = np.empty((k, self.n_out, self.n_in)) if order >= 1 else None
        hess = np.empty((k, self.n_out, self.n_in, self.n_in)) if order >= 2 else None
        st = _lib.lib().rtn_prepare(self.ctx_ptr, _arr(z), k, cols, order, _arr(f),
                                    _arr(jac) if jac is not None else None,
                                    _arr(hess) if hess is not None else None)
        raise_for_status(st)
        return BatchEval(f, jac, hess)

    def nonfinite(self, reset: bool = True) -> bool:
        """True when the last blocking call (or the device calls since the last
        reset) wrote a NaN/Inf output (rtn_ctx_nonfinite)."""
        flag = C.c_int()
        raise_for_status(_lib.lib().rtn_ctx_nonfinite(self.ctx_ptr, C.byref(flag), int(reset)))
        return bool(flag.value)

    def counters(self) -> tuple[int, int, int]:
        a, b, c = C.c_ulonglong(), C.c_ulonglong(), C.c_ulonglong()
        raise_for_status(_lib.lib().rtn_ctx_counters(self.ctx_ptr, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def close(self) -> None:
        L = _lib.lib()
        if self.ctx_ptr:
            L.rtn_ctx_free(self.ctx_ptr)
            self.ctx_ptr = C.c_void_p()
        if self.model_ptr:
            L.rtn_model_free(self.model_ptr)
            self.model_ptr = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# Entry points (proj/src/neural.cpp:300-327)

def mlp_batched_eval(m: MlpModel, z_rows, order: EvalOrder, counters: EvalCounters | None = None,
                     device: int = 0, precision: int = _lib.RTN_TF32) -> BatchEval:
    z_rows = np.atleast_2d(np.asarray(z_rows, dtype=np.float64))
    if counters is not None:
        counters.batched_calls += 1
        counters.batched_points += z_rows.shape[0]
    return m.engine(device, precision).prepare(z_rows, int(order))


def mlp_forward(m: MlpModel, z, counters: EvalCounters | None = None, **kw) -> np.ndarray:
    if counters is not None:
        counters.value_evals += 1
    z = np.asarray(z, dtype=np.float64)
    if z.shape != (m.input_dim(),):
        raise InputDomainError("mlp eval: feature dim does not match model input")
    return m.engine(**kw).prepare(z[None, :], 0).values[0]


def mlp_jacobian(m: MlpModel, z, counters: EvalCounters | None = None, **kw) -> np.ndarray:
    if counters is not None:
        counters.jacobian_evals += 1
    z = np.asarray(z, dtype=np.float64)
    if z.shape != (m.input_dim(),):
        raise InputDomainError("mlp eval: feature dim does not match model input")
    return m.engine(**kw).prepare(z[None, :], 1).jacobians[0]


def mlp_hessian(m: MlpModel, z, counters: EvalCounters | None = None, **kw) -> np.ndarray:
    if counters is not None:
        counters.hessian_evals += 1
    m.validate()
    z = np.asarray(z, dtype=np.float64)
    if z.shape != (m.input_dim(),):
        raise InputDomainError("mlp hessian: feature dim mismatch")
    return m.engine(**kw).prepare(z[None, :], 2).hessians[0]


# --------------------------------------------------------------------------
# Construction and files

def make_mlp(layer_sizes, activation: str = "tanh", variant: str = "full", seed: int = 0) -> MlpModel:
    """MakeMlp (neural.cpp:465-489) — std::mt19937_64 draws via librtn_mpc."""
    sizes = [int(s) for s in layer_sizes]
    if len(sizes) < 2:
        raise ConfigError("mlp: need at least input and output layers")
    if activation not in ACTIVATIONS:
        raise ConfigError(f"mlp: unknown activation {activation!r}")
    ws = [np.empty((sizes[l + 1], sizes[l])) for l in range(len(sizes) - 1)]
    bs = [np.empty(sizes[l + 1]) for l in range(len(sizes) - 1)]
    wp = (C.POINTER(C.c_double) * len(ws))(*[_arr(w) for w in ws])
    bp = (C.POINTER(C.c_double) * len(bs))(*[_arr(b) for b in bs])
    s32 = np.asarray(sizes, dtype=np.int32)
    if _lib.lib().rtn_make_mlp(s32.ctypes.data_as(C.POINTER(C.c_int)), len(sizes), int(seed) & (2**64 - 1),
                               wp, bp) != 0:
        raise ConfigError("mlp: bad layer sizes")
    m = MlpModel(sizes, ws, bs, activation, variant, np.zeros(sizes[0]), np.ones(sizes[0]),
                 np.zeros(sizes[-1]), np.ones(sizes[-1]), int(seed))
    m.validate()
    return m


def make_zero_network(depth: int, width: int, in_dim: int, out_dim: int, seed: int) -> MlpModel:
    """MakeZeroNetwork (proj/src/bench.cpp:25-36): MakeMlp tanh hidden layers
    with the last layer zeroed — the paper's §V timing trick:
    full network cost, zero residual, so the controller's behaviour is the
    nominal one. Outputs (f, J, H) are exactly zero."""
    if depth < 1 or width < 1 or in_dim < 1 or out_dim < 1:
        raise ConfigError("zero network: dimensions must be positive")
    m = make_mlp([in_dim] + [width] * depth + [out_dim], "tanh", "full", seed)
    m.weights[-1][:] = 0.0
    m.biases[-1][:] = 0.0
    return m


def synth_quad_nodes(seed: int, k: int) -> np.ndarray:
    """Quadrotor node rows z=[p q v ω u] (SURVEY §8d synthetic inputs)."""
    z = np.empty((k, 17))
    _lib.lib().rtn_synth_quad_nodes(int(seed), int(k), _arr(z))
    return z


def save_model(m: MlpModel, path: str) -> None:
    """RMLP v1 (tanh/relu, neural.cpp:685-718) or v2 (SiLU tag 2) + JSON sidecar."""
    m.validate()
    v2 = m.activation == "silu"
    var = m.input_variant.encode()
    with open(path, "wb") as fh:
        fh.write(b"RMLP")
        fh.write(struct.pack("<IBI", 2 if v2 else 1, ACTIVATIONS.index(m.activation), len(var)))
        fh.write(var)
        fh.write(struct.pack("<QI", int(m.seed), len(m.layer_sizes)))
        fh.write(struct.pack(f"<{len(m.layer_sizes)}I", *m.layer_sizes))
        for v in (m.in_mean, m.in_scale, m.out_mean, m.out_scale):
            fh.write(np.ascontiguousarray(v, dtype="<f8").tobytes())
        for w, b in zip(m.weights, m.biases):
            fh.write(np.ascontiguousarray(w, dtype="<f8").tobytes())
            fh.write(np.ascontiguousarray(b, dtype="<f8").tobytes())
    with open(path + ".json", "w") as fh:
        json.dump({"format": "RMLP", "version": 2 if v2 else 1, "activation": m.activation,
                   "input_variant": m.input_variant, "layer_sizes": m.layer_sizes, "arch": m.arch_name(),
                   "parameter_count": m.parameter_count(), "seed": int(m.seed)}, fh, indent=2)
        fh.write("\n")


def load_model(path: str) -> MlpModel:
    """RMLP reader (neural.cpp:720-755; v1 tag 0 → tanh, else relu; v2 tag 2 → silu)."""
    if not os.path.exists(path):
        raise ConfigError(f"model: cannot open '{path}'")
    with open(path, "rb") as fh:
        data = fh.read()
    off = 0

    def take(n):
        nonlocal off
        if off + n > len(data):
            raise ConfigError("unexpected end of file")
        b = data[off:off + n]
        off += n
        return b

    if take(4) != b"RMLP":
        raise ConfigError(f"model: '{path}' is not a model file")
    (version,) = struct.unpack("<I", take(4))
    if version not in (1, 2):
        raise ConfigError("model: unsupported version")
    (tag,) = struct.unpack("<B", take(1))
    if version == 1:
        act = "tanh" if tag == 0 else "relu"
    elif tag <= 2:
        act = ACTIVATIONS[tag]
    else:
        raise ConfigError("model: unknown activation tag")
    (n,) = struct.unpack("<I", take(4))
    variant = take(n).decode()
    seed, ns = struct.unpack("<QI", take(12))
    sizes = list(struct.unpack(f"<{ns}I", take(4 * ns)))
    if len(sizes) < 2:
        raise ConfigError("mlp: need at least input and output layers")

    def vec(k):
        return np.frombuffer(take(8 * k), dtype="<f8").astype(np.float64)

    in_mean, in_scale, out_mean, out_scale = vec(sizes[0]), vec(sizes[0]), vec(sizes[-1]), vec(sizes[-1])
    ws, bs = [], []
    for l in range(len(sizes) - 1):
        ws.append(vec(sizes[l + 1] * sizes[l]).reshape(sizes[l + 1], sizes[l]))
        bs.append(vec(sizes[l + 1]))
    m = MlpModel(sizes, ws, bs, act, variant, in_mean, in_scale, out_mean, out_scale, seed)
    m.validate()
    return m


def parse_arch(arch: str) -> list[int]:
    """'3x32' or '32,32,32' → hidden sizes (neural.cpp:757-776)."""
    if "x" in arch and "," not in arch:
        d, w = arch.split("x", 1)
        depth, width = int(d), int(w)
        if depth < 1 or width < 1:
            raise ConfigError(f"arch: bad depth/width in '{arch}'")
        return [width] * depth
    sizes = []
    for tok in arch.split(","):
        w = int(tok)
        if w < 1:
            raise ConfigError(f"arch: bad width in '{arch}'")
        sizes.append(w)
    if not sizes:
        raise ConfigError(f"arch: empty spec '{arch}'")
    return sizes


def flops_per_node(layer_sizes, order: int = 1) -> int:
    """Forward-mode algorithmic FLOPs per node: 2·rows·P_W."""
    n_in = layer_sizes[0]
    pw = sum(layer_sizes[l] * layer_sizes[l + 1] for l in range(len(layer_sizes) - 1))
    rows = 1 + n_in + (n_in * (n_in + 1) // 2 if order == 2 else 0)
    return 2 * rows * pw
