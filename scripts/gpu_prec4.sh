# 3xTF32 split accumulators (bf16x3 flag fix): probe, GPU suite, bench.
mkdir -p gpurun_out
timeout 300 python scripts/precision_probe.py 2>&1 | grep -v latency | tail -16
ORDER=2 PRECS=3xtf32,bf16x3 timeout 300 python scripts/precision_probe.py 2>&1 | grep pair | tail -10
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -5
timeout 900 python bench.py > gpurun_out/bench_prec4.json 2> gpurun_out/bench_prec4.err; echo "bench rc=$?"
