# Rows kernel round: GPU suite, bench line, ncu of the rows kernel at cfg4.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err; echo "bench rc=$?"
tail -2 gpurun_out/bench_r01e.err
RTN_KERNEL=rows timeout 600 ncu --set full --import-source on --clock-control none -k regex:rtn_rows_kernel -s 1 -c 1 -o gpurun_out/ncu_rows_final -f python scripts/ncu_target.py 256 5 silu 81920 2 > gpurun_out/ncu_rows_final.log 2>&1; tail -1 gpurun_out/ncu_rows_final.log
