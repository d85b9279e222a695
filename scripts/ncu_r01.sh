set -e
mkdir -p gpurun_out
python scripts/ncu_target.py 512 12 silu 409600 2 > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rtn_fused -s 1 -c 1 -o gpurun_out/prof_cfg5 python scripts/ncu_target.py 512 12 silu 409600 2 > gpurun_out/ncu_cfg5.log 2>&1
python scripts/ncu_target.py 256 5 silu 81920 2 > gpurun_out/plain4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rtn_fused -s 1 -c 1 -o gpurun_out/prof_cfg4 python scripts/ncu_target.py 256 5 silu 81920 2 > gpurun_out/ncu_cfg4.log 2>&1
ls -la gpurun_out
