"""CPU tests of the drop-in boundary: librtn_mpc.so loads, exports exactly the
entry points include/rtn_mpc.h declares, and validates arguments (mapping the
reference's exceptions to status codes) before touching a device."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2203_07747_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rtn_mpc.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(rtn_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(L, n), n
    assert set(_lib.EXPORTS) <= set(names)


def test_status_codes_match_header():
    src = open(HEADER).read()
    vals = dict(re.findall(r"(RTN_E\w+|RTN_OK)\s*=\s*(\d+)", src))
    assert int(vals["RTN_OK"]) == _lib.RTN_OK
    assert int(vals["RTN_ECONFIG"]) == _lib.RTN_ECONFIG
    assert int(vals["RTN_EDOMAIN"]) == _lib.RTN_EDOMAIN
    assert int(vals["RTN_EUNSUPPORTED"]) == _lib.RTN_EUNSUPPORTED
    assert int(vals["RTN_ECUDA"]) == _lib.RTN_ECUDA


def _from_arrays(sizes, act=2, in_scale=None):
    L = _lib.lib()
    ws = [np.zeros((sizes[l + 1], sizes[l])) for l in range(len(sizes) - 1)]
    bs = [np.zeros(sizes[l + 1]) for l in range(len(sizes) - 1)]
    dp = C.POINTER(C.c_double)
    wp = (dp * len(ws))(*[w.ctypes.data_as(dp) for w in ws])
    bp = (dp * len(bs))(*[b.ctypes.data_as(dp) for b in bs])
    norm = [np.zeros(sizes[0]), np.ones(sizes[0]) if in_scale is None else in_scale, np.zeros(sizes[-1]),
            np.ones(sizes[-1])]
    s = np.asarray(sizes, dtype=np.int32)
    out = C.c_void_p()
    st = L.rtn_model_from_arrays(s.ctypes.data_as(C.POINTER(C.c_int)), len(sizes), act, wp, bp,
                                 *[v.ctypes.data_as(dp) for v in norm], 0, 0, C.byref(out))
    return st, out


def test_config_errors_before_device():
    # proj/src/neural.cpp:283-298 → ConfigError → RTN_ECONFIG
    st, _ = _from_arrays([17, 64, 6], in_scale=np.zeros(17))
    assert st == _lib.RTN_ECONFIG
    assert "strictly positive" in _lib.last_error()
    st, _ = _from_arrays([17, 64, 6], act=9)
    assert st == _lib.RTN_ECONFIG


def test_unsupported_shapes_before_device():
    st, _ = _from_arrays([17, 1024, 6])       # hidden width > 512
    assert st == _lib.RTN_EUNSUPPORTED
    st, _ = _from_arrays([17, 64, 32])         # n_out > 16
    assert st == _lib.RTN_EUNSUPPORTED


def test_rmlp_load_errors(tmp_path):
    L = _lib.lib()
    out = C.c_void_p()
    assert L.rtn_model_load_rmlp(b"/nonexistent.rmlp", 0, 0, C.byref(out)) == _lib.RTN_ECONFIG
    p = tmp_path / "bad.rmlp"
    p.write_bytes(b"NOPE")
    assert L.rtn_model_load_rmlp(str(p).encode(), 0, 0, C.byref(out)) == _lib.RTN_ECONFIG


def test_no_cpu_fallback_without_device():
    """Valid models fail loudly with RTN_ECUDA on a machine without a B200
    (there is no CPU fallback path)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("device present")
    except Exception:
        pass
    st, _ = _from_arrays([17, 64, 64, 6])
    assert st == _lib.RTN_ECUDA
