# Round-2 profiles: launch list of the bench step, then ncu --set full of the
# cfg5 TF32 throughput kernel, its bf16 variant and the cfg3 quad latency kernel.
set -x
mkdir -p gpurun_out
python bench.py --steps 2 --warmup 3 --no-cpu --no-latency --no-modes --no-blocks > gpurun_out/plain_bench.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu --no-latency --no-modes --no-blocks > gpurun_out/ncu_launch.log 2>&1
python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rtn_pair -s 1 -c 1 -o gpurun_out/prof_r02_pair -f \
    python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/ncu_pair.log 2>&1
python scripts/ncu_target.py 512 12 silu 102400 2 bf16 > gpurun_out/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rtn_pair -s 1 -c 1 -o gpurun_out/prof_r02_pair_bf16 -f \
    python scripts/ncu_target.py 512 12 silu 102400 2 bf16 > gpurun_out/ncu_pair_bf16.log 2>&1
python scripts/ncu_target.py 512 12 silu 20 4 > gpurun_out/plainq.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rtn_quad -s 2 -c 1 -o gpurun_out/prof_r02_quad -f \
    python scripts/ncu_target.py 512 12 silu 20 4 > gpurun_out/ncu_quad.log 2>&1
ls -la gpurun_out
