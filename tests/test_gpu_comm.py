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
