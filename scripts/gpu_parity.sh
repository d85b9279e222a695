nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "cfg1" 2>&1 | tail -30
timeout 400 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -30
