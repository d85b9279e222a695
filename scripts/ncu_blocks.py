"""ncu target: one warm + one profiled rtn_build_qp_device launch (8192 x 50 nodes)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
from paper_2203_07747_b200 import _lib, make_mlp, qp
from paper_2203_07747_b200.errors import raise_for_status
n_inst, n = int(os.environ.get("NI", 8192)), 50
k = n_inst * n
xs, us, rx, ru = bench._quad_iterate(np, n_inst, n, 1)
rng = np.random.default_rng(2)
z0 = np.concatenate([xs[:, :n], us], axis=-1).reshape(k, 17)
fb, jac = rng.normal(0, .5, (k, 6)), rng.normal(0, .1, (k, 6, 17))
d = [torch.from_numpy(np.ascontiguousarray(a)).cuda() for a in (xs, us, rx, ru, z0, fb, jac)]
outs = [torch.empty(s, dtype=torch.float64, device="cuda") for s in
        [(k, 13, 13), (k, 13, 4), (k, 13), (n_inst, n + 1, 13), (k, 4), (n_inst, n + 1, 13), (k, 4), (k, 4), (k, 4)]]
eng = make_mlp([17, 64, 6], "silu", "full", 1).engine()
eng._ensure(64, 1)
p, cfg = qp.QuadParams().to_c(), qp.OcpConfig(horizon=n, dt=0.02).to_c()
it = _lib.IterateC(*[t.data_ptr() for t in d[:4]])
ap = _lib.ApproxC(d[4].data_ptr(), d[5].data_ptr(), d[6].data_ptr(), None)
oc = _lib.QpBlocksC(*[t.data_ptr() for t in outs])
L = _lib.lib()
for _ in range(int(os.environ.get("REPS", 2))):
    raise_for_status(L.rtn_build_qp_device(eng.ctx_ptr, C.byref(p), C.byref(cfg), n_inst, C.byref(it), C.byref(ap), C.byref(oc)))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
st = torch.cuda.current_stream()
raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
e0.record()
raise_for_status(L.rtn_build_qp_device(eng.ctx_ptr, C.byref(p), C.byref(cfg), n_inst, C.byref(it), C.byref(ap), C.byref(oc)))
e1.record(); e1.synchronize()
print("blocks ms", e0.elapsed_time(e1), "nodes", k, "ns/node", e0.elapsed_time(e1) * 1e6 / k)
