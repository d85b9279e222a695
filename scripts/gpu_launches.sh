timeout 300 python bench.py --steps 2 --warmup 3 --no-latency --no-cpu --no-modes --no-blocks > gpurun_out/b_plain.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --no-latency --no-cpu --no-modes --no-blocks > gpurun_out/ncu_bench.log 2>&1
tail -2 gpurun_out/launches.csv
