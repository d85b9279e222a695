timeout 300 python -m pytest tests/test_gpu_blocks.py -q -x 2>&1 | tail -1
RTN_ZEROCOPY=0 timeout 300 python -m pytest tests/test_gpu_blocks.py -q -x 2>&1 | tail -1
for zc in 0 1; do RTN_ZEROCOPY=$zc timeout 300 python scripts/blocks_probe.py 2>&1 | grep -E "p50_us" | tr '\n' ' '; echo " zc=$zc"; done
