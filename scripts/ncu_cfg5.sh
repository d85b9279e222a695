set -e
mkdir -p gpurun_out
python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:rtn_fused -s 1 -c 1 -o gpurun_out/prof_cfg5b -f python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/ncu_cfg5.log 2>&1
