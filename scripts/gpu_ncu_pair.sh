timeout 120 python scripts/ncu_target.py 512 12 silu 102400 2 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rtn_pair_kernel -s 1 -c 1 -o gpurun_out/ncu_pair_cfg5 -f python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/ncu_pair.log 2>&1; tail -1 gpurun_out/ncu_pair.log
