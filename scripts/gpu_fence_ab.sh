for r in 1 2; do
for dbg in 0 256; do echo "dbg=$dbg (256 = cluster fence everywhere)"; RTN_DEBUG=$dbg timeout 200 python scripts/perf_probe.py 0 2>&1 | grep -E "K=409600|K=81920"; done
done
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_precision.py -q 2>&1 | tail -1
