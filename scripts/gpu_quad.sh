L=12 KS=1,2,7,20,74 timeout 120 python scripts/quad_smoke.py; echo rc=$?
for qd in 0 1 0 1; do RTN_QUAD=$qd timeout 300 python - <<'PY'
import os, sys
sys.path.insert(0, os.getcwd())
import torch, bench
r1 = bench.latency(torch, bench.SIZES, bench.SEED, 20)
print("quad", os.environ["RTN_QUAD"], "cfg3 p50 %.1f p99 %.1f dev %.1f" % (r1["p50_us"], r1["p99_us"], r1["device_p50_us"]))
PY
done
