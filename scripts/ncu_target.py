"""Small single-purpose driver for ncu: N launches of the fused kernel on one
BASELINE shape (device-resident inputs).

usage: python scripts/ncu_target.py <width> <depth> <act> <K> [launches] [precision]
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2203_07747_b200 import _lib, make_mlp, synth_quad_nodes  # noqa: E402
from paper_2203_07747_b200.errors import raise_for_status  # noqa: E402

width, depth, act, k = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
launches = int(sys.argv[5]) if len(sys.argv) > 5 else 2
prec = (_lib.PRECISIONS.get(sys.argv[6]) if sys.argv[6] in _lib.PRECISIONS else int(sys.argv[6])) if len(sys.argv) > 6 else 0
sizes = [17] + [width] * depth + [6]
m = make_mlp(sizes, act, "full", 1000 * depth + width)
eng = m.engine(precision=prec)
eng._ensure(k, 1)
L = _lib.lib()
st = torch.cuda.Stream()
torch.cuda.set_stream(st)
raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
z = torch.from_numpy(synth_quad_nodes(2203, k)).cuda()
f = torch.empty((k, 6), dtype=torch.float64, device="cuda")
j = torch.empty((k, 6, 17), dtype=torch.float64, device="cuda")
for _ in range(launches):
    raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(), j.data_ptr(), None))
torch.cuda.synchronize()
print("ok", float(f.abs().sum()), float(j.abs().sum()))
