timeout 60 python scripts/trace_rows.py 2>&1 | tail -8
RTN_KERNEL=rows timeout 90 python -m pytest tests/test_gpu_parity.py -q -x -k "rows" 2>&1 | tail -2
timeout 120 python scripts/perf_probe.py 2>&1 | sed -n 1,2p
RTN_DEBUG=128 timeout 60 python scripts/perf_probe.py 2>&1 | sed -n 2,2p
