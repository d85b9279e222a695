# 3xTF32 split main accumulators: precision probe (orders 1, 2), GPU suite, bench.
mkdir -p gpurun_out
PRECS=3xtf32 timeout 300 python scripts/precision_probe.py 2>&1 | tail -8
ORDER=2 PRECS=3xtf32 timeout 300 python scripts/precision_probe.py 2>&1 | tail -8
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_prec3.json 2> gpurun_out/bench_prec3.err; echo "bench rc=$?"
