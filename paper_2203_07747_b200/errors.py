"""Error classes of the reference (proj/include/resmpc/errors.hpp:9-22) and the
C-ABI status → exception mapping (include/rtn_mpc.h)."""
from __future__ import annotations


class ConfigError(RuntimeError):
    """Bad file contents, incompatible metadata, invalid configuration values."""


class InputDomainError(ValueError):
    """Caller handed a value outside the documented input domain."""


class UnsupportedError(RuntimeError):
    """Operation not defined for this configuration (e.g. Hessians of relu nets)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL failure underneath the C-ABI."""


def raise_for_status(status: int) -> None:
    if status == 0:
        return
    from . import _lib
    msg = _lib.last_error()
    # 6: std::runtime_error of BuildQp ("build qp: node k: ...", sqp_rti.cpp:134-138)
    cls = {1: ConfigError, 2: InputDomainError, 3: UnsupportedError, 6: RuntimeError}.get(status, DeviceError)
    raise cls(msg)
