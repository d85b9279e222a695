"""cfg5-shape device time of the throughput kernel under the RTN_DEBUG isolation
switches (rtn_pair.cuh): 0 full, 4 epilogue math/stores skipped (publish only),
8 peer-side stores made local (DSMEM cost), 128 weight stream + MMAs only.
Usage: RTN_DEBUG=<n> [JMODE=1: reverse mode] python scripts/pair_isolate.py [K]"""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2203_07747_b200 import _lib, flops_per_node, make_mlp, synth_quad_nodes  # noqa: E402
from paper_2203_07747_b200.errors import raise_for_status  # noqa: E402

sizes = [17] + [int(os.environ.get("WIDTH", "512"))] * int(os.environ.get("DEPTH", "12")) + [int(os.environ.get("NOUT", "6"))]
k = int(sys.argv[1]) if len(sys.argv) > 1 else 409600
prec = _lib.PRECISIONS.get(os.environ.get("PREC", "tf32"), None)
prec = int(os.environ.get("PREC")) if prec is None else prec  # a name (tf32, bf16, ...) or the enum value
m = make_mlp(sizes, "silu", "full", 12512)
eng = m.engine(precision=prec, jacobian_mode=int(os.environ.get("JMODE", "0")))
eng._ensure(k, 1)
L = _lib.lib()
z = torch.from_numpy(synth_quad_nodes(2203, k)).cuda()
f = torch.empty((k, sizes[-1]), dtype=torch.float64, device="cuda")
j = torch.empty((k, sizes[-1], 17), dtype=torch.float64, device="cuda")
st = torch.cuda.Stream()
raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
run = lambda: raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(), j.data_ptr(), None))
with torch.cuda.stream(st):
    for _ in range(2):
        run()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        run()
        e1.record(st)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
t = float(np.median(ts))
tf = k * flops_per_node(sizes) / (t * 1e-3) / 1e12
print(f"dbg={os.environ.get('RTN_DEBUG', '0')} prec={prec} K={k} {sizes[1]}x{len(sizes) - 2}: {t:.2f} ms  "
      f"{k / t / 1e3:.2f} M node-lin/s  {tf:.1f} TFLOP/s", flush=True)
