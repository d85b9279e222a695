for d in 0 16 4; do RTN_DEBUG=$d python scripts/pair_isolate.py 409600; done > gpurun_out/isolate.txt 2>&1
RTN_TRACE=3 python scripts/trace_tput.py 409600 > gpurun_out/trace_tput.txt 2>&1
cat gpurun_out/isolate.txt; head -12 gpurun_out/trace_tput.txt
