timeout 600 python -m pytest tests -q -m gpu 2>&1 | tail -4
timeout 900 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json
