"""Quick device-time probe of the fused kernel on the BASELINE shapes."""
import ctypes as C
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2203_07747_b200 import _lib, make_mlp, synth_quad_nodes, flops_per_node  # noqa: E402
from paper_2203_07747_b200.errors import raise_for_status  # noqa: E402


def probe(sizes, act, k, reps=5, prec=0):
    m = make_mlp(sizes, act, "full", 1000 * (len(sizes) - 2) + sizes[1])
    eng = m.engine(precision=prec)
    eng._ensure(k, 1)
    L = _lib.lib()
    z = torch.from_numpy(synth_quad_nodes(2203, k)).cuda()
    f = torch.empty((k, 6), dtype=torch.float64, device="cuda")
    j = torch.empty((k, 6, 17), dtype=torch.float64, device="cuda")
    st = torch.cuda.Stream()
    torch.cuda.set_stream(st)
    raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
    for _ in range(2):
        raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(), j.data_ptr(), None))
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(), j.data_ptr(), None))
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = float(np.median(ts))
    fl = flops_per_node(sizes) * k
    print(f"prec {prec} {sizes[1]}x{len(sizes)-2} {act} K={k}: {t:.3f} ms  {k/t*1e3/1e6:.2f} M nodes/s  {fl/t/1e9:.1f} TFLOP/s", flush=True)


if __name__ == "__main__":
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device="cuda")
    b = torch.randn(8192, 8192, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); a @ b; e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"cuBLAS tf32 8192^3: {2*8192**3/best/1e9:.1f} TFLOP/s", flush=True)
    precs = [int(x) for x in sys.argv[1:]] or [0]
    for pr in precs:
        probe([17] + [256] * 5 + [6], "silu", 81920, prec=pr)
        probe([17] + [512] * 12 + [6], "silu", 20, prec=pr)
        probe([17] + [256] * 5 + [6], "silu", 20, prec=pr)
        probe([17] + [512] * 12 + [6], "silu", 3276800 // 8, prec=pr)
    if precs == [0]:
        probe([17] + [512] * 12 + [6], "silu", 3276800, reps=3)
