for d in 0 4 8 128; do RTN_DEBUG=$d python scripts/pair_isolate.py 409600; done > gpurun_out/isolate.txt 2>&1
RTN_TRACE=3 python scripts/trace_tput.py 409600 > gpurun_out/trace_tput.txt 2>&1
cat gpurun_out/isolate.txt gpurun_out/trace_tput.txt
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1
tail -n 15 gpurun_out/pytest_gpu.txt
