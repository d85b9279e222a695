for zc in 0 1 0 1; do RTN_ZEROCOPY=$zc timeout 300 python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import torch, bench
r1 = bench.latency(torch, bench.SIZES, bench.SEED, 20)
r2 = bench.latency(torch, bench.SIZES, bench.SEED, 20, steps=300, order=2)
print("zc", os.environ["RTN_ZEROCOPY"], "o1 p50 %.1f p99 %.1f | o2 p50 %.1f p99 %.1f" % (r1["p50_us"], r1["p99_us"], r2["p50_us"], r2["p99_us"]))
PY
done
RTN_ZEROCOPY=1 timeout 300 python -m pytest tests/test_gpu_api.py tests/test_gpu_order2.py -q -x 2>&1 | tail -1
