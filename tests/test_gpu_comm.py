"""The multi-GPU C-ABI entry (include/rtn_mpc.h rtn_comm_*, rtn_prepare_partitioned*;
csrc/rtn_comm.cu) on the one GPU of the test box: a single-rank NCCL communicator,
so the root's receives come from its own chunked sends. The partition/gather
bookkeeping across several ranks is covered on CPU by tests/test_sharding.py
(gloo, world size 2) through the same chunking rule (sharding.chunk_bounds)."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
from paper_2203_07747_b200 import _lib
from paper_2203_07747_b200.errors import raise_for_status

pytestmark = pytest.mark.gpu


def _engine(sizes, act="silu", gain=2.0):
    om = oracle.OracleModel.random_net(sizes, act, 11, True)
    for l, (w, b) in enumerate(om.layers()):
        if l < len(sizes) - 2:
            om.set_layer(l, w * gain, b)
    return om, oracle.to_product_model(om).engine()


def _comm():
    L = _lib.lib()
    uid = C.create_string_buffer(128)
    raise_for_status(L.rtn_comm_unique_id(uid))
    cm = C.c_void_p()
    raise_for_status(L.rtn_comm_create(uid, 1, 0, 0, C.byref(cm)))
    return cm


def test_partitioned_host_entry_matches_prepare():
    L = _lib.lib()
    om, eng = _engine([17] + [256] * 3 + [6])
    k = 5000
    z = oracle.quad_nodes(3, k)
    eng._ensure(k, 1)
    ref = eng.prepare(z, 1)
    cm = _comm()
    f = np.empty((k, 6))
    j = np.empty((k, 6, 17))
    raise_for_status(L.rtn_prepare_partitioned(eng.ctx_ptr, cm, z.ctypes.data, k, 17, 1, 0, f.ctypes.data,
                                               j.ctypes.data))
    assert np.array_equal(f, ref.values) and np.array_equal(j, ref.jacobians)
    calls, points, _ = eng.counters()
    assert points >= 2 * k
    # order 2 is not gathered (Hessians stay on their rank)
    assert L.rtn_prepare_partitioned(eng.ctx_ptr, cm, z.ctypes.data, k, 17, 2, 0, f.ctypes.data,
                                     j.ctypes.data) == _lib.RTN_EUNSUPPORTED
    # bad root
    assert L.rtn_prepare_partitioned(eng.ctx_ptr, cm, z.ctypes.data, k, 17, 1, 1, f.ctypes.data,
                                     j.ctypes.data) == _lib.RTN_ECONFIG
    L.rtn_comm_free(cm)


@pytest.mark.parametrize("chunks", [1, 3, 8])
def test_partitioned_device_entry_chunked(chunks):
    """Chunk i's send/recv overlaps chunk i+1's kernel; the gathered rows equal
    the rank's own outputs and the fp64 oracle."""
    L = _lib.lib()
    om, eng = _engine([17] + [512] * 4 + [6])
    k = 3001
    z = oracle.quad_nodes(4, k)
    eng._ensure(k, 1)
    dz = torch.from_numpy(z).cuda()
    df = torch.empty((k, 6), dtype=torch.float64, device="cuda")
    dj = torch.empty((k, 6, 17), dtype=torch.float64, device="cuda")
    fa = torch.full((k, 6), np.nan, dtype=torch.float64, device="cuda")
    ja = torch.full((k, 6, 17), np.nan, dtype=torch.float64, device="cuda")
    cm = _comm()
    raise_for_status(L.rtn_prepare_partitioned_device(eng.ctx_ptr, cm, dz.data_ptr(), k, 1, df.data_ptr(),
                                                      dj.data_ptr(), 0, fa.data_ptr(), ja.data_ptr(), chunks))
    raise_for_status(L.rtn_ctx_synchronize(eng.ctx_ptr))
    assert torch.equal(fa, df) and torch.equal(ja, dj)
    f, j, _ = om.batched_eval(z[::37], 1)
    assert oracle.max_node_rel_error(fa.cpu().numpy()[::37], f) < 1e-3
    assert oracle.max_node_rel_error(ja.cpu().numpy()[::37], j) < 1e-3
    L.rtn_comm_free(cm)


def test_partitioned_p2p_single_rank():
    """Peer-store gather entry on one rank: the bound root outputs (here the
    rank's own, inside a larger allocation) receive the kernel's stores
    directly; bitwise equal to rtn_prepare_device."""
    L = _lib.lib()
    om, eng = _engine([17] + [512] * 4 + [6])
    k = 2501
    z = oracle.quad_nodes(6, k)
    eng._ensure(k, 1)
    dz = torch.from_numpy(z).cuda()
    df = torch.empty((k, 6), dtype=torch.float64, device="cuda")
    dj = torch.empty((k, 6, 17), dtype=torch.float64, device="cuda")
    raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, dz.data_ptr(), k, 1, df.data_ptr(), dj.data_ptr(), None))
    raise_for_status(L.rtn_ctx_synchronize(eng.ctx_ptr))
    big_f = torch.full((k + 64, 6), np.nan, dtype=torch.float64, device="cuda")
    big_j = torch.full((k + 64, 6, 17), np.nan, dtype=torch.float64, device="cuda")
    fa, ja = big_f[32:], big_j[32:]  # pointers inside the allocations
    cm = _comm()
    assert L.rtn_prepare_partitioned_p2p(eng.ctx_ptr, cm, dz.data_ptr(), k, 1) == _lib.RTN_ECONFIG  # not bound
    raise_for_status(L.rtn_comm_bind_root_outputs(cm, 0, fa.data_ptr(), ja.data_ptr(), k + 32))
    raise_for_status(L.rtn_prepare_partitioned_p2p(eng.ctx_ptr, cm, dz.data_ptr(), k, 1))
    raise_for_status(L.rtn_ctx_synchronize(eng.ctx_ptr))
    assert torch.equal(fa[:k], df) and torch.equal(ja[:k], dj)
    assert torch.isnan(big_f[:32]).all() and torch.isnan(fa[k:]).all()  # nothing outside the rank's rows
    assert L.rtn_prepare_partitioned_p2p(eng.ctx_ptr, cm, dz.data_ptr(), k, 2) == _lib.RTN_EUNSUPPORTED
    raise_for_status(L.rtn_comm_bind_root_outputs(cm, 0, fa.data_ptr(), ja.data_ptr(), k - 1))
    assert L.rtn_prepare_partitioned_p2p(eng.ctx_ptr, cm, dz.data_ptr(), k, 1) == _lib.RTN_ECONFIG  # rows exceed
    L.rtn_comm_free(cm)


_CHILD = r"""
import ctypes as C, sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_2203_07747_b200 import _lib
from paper_2203_07747_b200.errors import raise_for_status
hf, hj, lo, hi = bytes.fromhex(sys.argv[1]), bytes.fromhex(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
L = _lib.lib()
om = oracle.OracleModel.random_net([17] + [512] * 4 + [6], "silu", 11, True)
for l, (w, b) in enumerate(om.layers()):
    if l < 4:
        om.set_layer(l, w * 2.0, b)
eng = oracle.to_product_model(om).engine()
eng._ensure(hi - lo, 1)
z = torch.from_numpy(oracle.quad_nodes(7, hi)[lo:]).cuda()
pf, pj = C.c_void_p(), C.c_void_p()
raise_for_status(L.rtn_ipc_import(hf, 0, C.byref(pf)))
raise_for_status(L.rtn_ipc_import(hj, 0, C.byref(pj)))
raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), hi - lo, 1, pf.value + lo * 6 * 8,
                                      pj.value + lo * 6 * 17 * 8, None))
raise_for_status(L.rtn_ctx_synchronize(eng.ctx_ptr))
raise_for_status(L.rtn_ipc_release(pf))
raise_for_status(L.rtn_ipc_release(pj))
print("child ok")
"""


def test_ipc_peer_store_from_another_process():
    """The peer-store mechanics across processes: a second process maps this
    process's output buffers (rtn_ipc_export / rtn_ipc_import) and its kernel
    stores its rows into them; the assembled result equals one rtn_prepare over
    all rows, bitwise. (One GPU here, so the 'peer' is the same device; on a
    B200 box the same stores cross NVLink.)"""
    import os
    import subprocess
    import sys
    L = _lib.lib()
    om, eng = _engine([17] + [512] * 4 + [6])
    k, split = 3000, 1300
    z = oracle.quad_nodes(7, k)
    eng._ensure(k, 1)
    ref = eng.prepare(z, 1)
    fa = torch.full((k, 6), np.nan, dtype=torch.float64, device="cuda")
    ja = torch.full((k, 6, 17), np.nan, dtype=torch.float64, device="cuda")
    dz = torch.from_numpy(z[:split]).cuda()
    raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, dz.data_ptr(), split, 1, fa.data_ptr(), ja.data_ptr(), None))
    raise_for_status(L.rtn_ctx_synchronize(eng.ctx_ptr))
    hf, hj = C.create_string_buffer(72), C.create_string_buffer(72)
    raise_for_status(L.rtn_ipc_export(fa.data_ptr(), hf))
    raise_for_status(L.rtn_ipc_export(ja.data_ptr(), hj))
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _CHILD, hf.raw.hex(), hj.raw.hex(), str(split), str(k)], cwd=root,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "child ok" in r.stdout, r.stderr[-2000:]
    torch.cuda.synchronize()
    assert np.array_equal(fa.cpu().numpy(), ref.values)
    assert np.array_equal(ja.cpu().numpy(), ref.jacobians)
