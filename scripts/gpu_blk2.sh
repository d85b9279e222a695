timeout 300 python -m pytest tests/test_gpu_blocks.py -x -q 2>&1 | tail -2
NI=65536 REPS=2 timeout 120 python scripts/ncu_blocks.py
timeout 300 python scripts/blocks_probe.py 2>&1 | grep -E '"value"|achieved|frac|p50_us|p99_us'
ORDER=2 REPS=20 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cycle2_launches.csv python scripts/cycle_probe.py > /dev/null 2>&1
tail -3 gpurun_out/cycle2_launches.csv | cut -d, -f5,15
