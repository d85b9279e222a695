timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 300 python - <<'PY'
import sys, json; sys.path.insert(0,'.')
import torch, bench
print(json.dumps({"cfg3": bench.latency(torch, bench.SIZES, bench.SEED, 20), "cfg2": bench.latency(torch, [17]+[256]*5+[6], 5256, 20)}))
PY
