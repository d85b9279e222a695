# 3xTF32 on the 4-CTA latency kernel: parity, precision, latency.
timeout 120 python -m pytest tests/test_gpu_parity.py -q -x -k "quad" 2>&1 | tail -2
timeout 300 python -m pytest tests/test_gpu_precision.py -q -x 2>&1 | tail -3
PRECS=3xtf32 timeout 300 python scripts/precision_probe.py 2>&1 | grep latency | head -5
timeout 200 python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import bench
S = [17] + [512] * 12 + [6]
for prec, name in ((1, "3xtf32"), (2, "bf16x3")):
    r = bench.latency(torch, S, 12512, 20, steps=300, precision=prec)
    print(f"{name} cfg3 latency: p50 {r['p50_us']:.1f} p99 {r['p99_us']:.1f} device p50 {r['device_p50_us']:.1f}")
PY
