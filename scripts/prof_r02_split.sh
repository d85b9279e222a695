# Round-2 profiles of the split kernel: launch list of the bench step (the cfg5
# TF32 default is now rtn_split_kernel), then ncu --set full of one launch.
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu --no-latency --no-modes --no-blocks > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02_split.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-latency --no-modes --no-blocks > gpurun_out/ncu_launch.log 2>&1
python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rtn_split -s 1 -c 1 -o gpurun_out/prof_r02_split -f \
    python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/ncu_split.log 2>&1
ls -la gpurun_out | tail -5
