set -e
timeout 120 python scripts/ncu_blocks.py
timeout 600 ncu --set full --import-source on --clock-control none -k regex:QpBlocksKernel -c 1 -o gpurun_out/ncu_blocks -f python scripts/ncu_blocks.py > gpurun_out/ncu_blocks.log 2>&1
tail -3 gpurun_out/ncu_blocks.log
