# 3xTF32 correction accumulator: precision probe (orders 1, 2), split-mode tests, bench.
mkdir -p gpurun_out
timeout 300 python scripts/precision_probe.py 2>&1 | grep -v "^tf32" | tail -30
ORDER=2 timeout 300 python scripts/precision_probe.py 2>&1 | grep 3xtf32 | tail -10
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_prec2.json 2> gpurun_out/bench_prec2.err; echo "bench rc=$?"
