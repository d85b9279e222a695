"""Per-layer event timeline of pair 0 (RTN_TRACE) for a latency-mode call."""
import ctypes as C, os, sys
os.environ["RTN_TRACE"] = "1"
sys.path.insert(0, ".")
import numpy as np
from paper_2203_07747_b200 import _lib, make_mlp, synth_quad_nodes, mlp_batched_eval, EvalOrder
sizes = [17] + [512] * 12 + [6] if len(sys.argv) < 2 else [17] + [int(sys.argv[1])] * int(sys.argv[2]) + [6]
k = int(sys.argv[3]) if len(sys.argv) > 3 else 20
m = make_mlp(sizes, "silu", "full", 12512)
z = synth_quad_nodes(7, k)
for _ in range(5):
    mlp_batched_eval(m, z, EvalOrder.JACOBIAN)
L = _lib.lib()
buf = (C.c_ulonglong * 256)()
L.rtn_debug_trace(buf, 256)
t = np.array(buf, dtype=np.float64)
t0 = min(x for x in (t[196], t[197]) if x > 0)
rel = lambda x: (x - t0) / 1e3 if x > 0 else float("nan")
print(f"kernel start CTA0 {rel(t[196]):7.2f} us CTA1 {rel(t[197]):7.2f}; layer0 done CTA0 {rel(t[192]):7.2f} CTA1 {rel(t[193]):7.2f}")
H = len(sizes) - 3
nmb = (max(sizes[1:-1]) + 255) // 256
for l in range(H):
    for mb in range(nmb):
        i = (l * 2 + mb)
        e0 = [rel(t[64 + i * 3 + q]) for q in range(3)]
        e1 = [rel(t[128 + i * 3 + q]) for q in range(3)]
        print(f"L{l+1} mb{mb}: mma {rel(t[i*2]):7.2f}-{rel(t[i*2+1]):7.2f} | CTA0 tfull {e0[0]:7.2f} infree {e0[1]:7.2f} pub {e0[2]:7.2f} | CTA1 tfull {e1[0]:7.2f} infree {e1[1]:7.2f} pub {e1[2]:7.2f}")
print(f"output tmem_last CTA0 {rel(t[194]):7.2f} CTA1 {rel(t[195]):7.2f}")
print("layer 2 mb1 per stage (us, rel): producer-issue | mma after full-wait | after mma issue")
for c in range(16):
    print(f"  c={c:2d}  {rel(t[200+c]):7.3f} | {rel(t[216+c]):7.3f} | {rel(t[232+c]):7.3f}")
dt_ns = t[252] - t[196]
dcyc = t[254] - t[250]
print(f"CTA0 kernel span {dt_ns/1e3:.2f} us, {dcyc:.0f} cycles -> SM clock {dcyc/dt_ns*1e3:.0f} MHz")
