# rows kernel (activations as A in TMEM): focused parity, then the suite, then cfg4 numbers.
mkdir -p gpurun_out
timeout 180 python -m pytest tests/test_gpu_parity.py -q -x -k "rows" 2>&1 | tail -15
timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -5
timeout 300 python scripts/perf_probe.py 2>&1 | tail -20
