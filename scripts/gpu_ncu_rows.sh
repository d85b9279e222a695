# ncu --set full of the rows kernel at cfg4 (one launch after warm-up).
mkdir -p gpurun_out
RTN_KERNEL=rows timeout 60 python scripts/ncu_target.py 256 5 silu 81920 2 || exit 1
RTN_KERNEL=rows timeout 600 ncu --set full --import-source on --clock-control none -k regex:rtn_rows_kernel -s 1 -c 1 -o gpurun_out/ncu_rows -f python scripts/ncu_target.py 256 5 silu 81920 2 > gpurun_out/ncu_rows.log 2>&1; tail -2 gpurun_out/ncu_rows.log
