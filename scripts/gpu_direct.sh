timeout 300 python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
for rep in range(2):
    r1 = bench.latency(torch, bench.SIZES, bench.SEED, 20)
    r2 = bench.latency(torch, bench.SIZES, bench.SEED, 20, steps=300, order=2)
    r3 = bench.latency(torch, [17] + [256] * 5 + [6], 5256, 20)
    print("o1 p50 %.1f p99 %.1f | o2 p50 %.1f p99 %.1f dev %.1f | cfg2 %.1f" % (r1["p50_us"], r1["p99_us"], r2["p50_us"], r2["p99_us"], r2["device_p50_us"], r3["p50_us"]))
PY
timeout 300 python -m pytest tests/test_gpu_api.py tests/test_gpu_order2.py tests/test_gpu_parity.py -q 2>&1 | tail -1
