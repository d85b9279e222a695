timeout 300 python scripts/precision_probe.py 2>&1 | tail -30
timeout 300 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
