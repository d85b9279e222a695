set -e
mkdir -p gpurun_out
# launch list of the bench command (cold-cache, serialised per-launch times)
python bench.py --steps 2 --warmup 3 --no-cpu --no-latency > gpurun_out/plain_bench.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-latency > gpurun_out/ncu_launch.log 2>&1
# full capture of the top kernel on a smaller batch
python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/plain.log 2>&1
RTN_KERNEL=pair ncu --set full --clock-control none --import-source on -k regex:rtn_pair -s 1 -c 1 -o gpurun_out/prof_r01 -f python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/ncu_full.log 2>&1
