NI=65536 REPS=2 timeout 120 python scripts/ncu_blocks.py
NI=1 REPS=5 timeout 120 python scripts/ncu_blocks.py
timeout 300 python -m pytest tests/test_gpu_blocks.py -x -q 2>&1 | tail -2
timeout 300 python scripts/blocks_probe.py 2>&1 | grep -E '"value"|achieved|frac|p50_us|p99_us' 
