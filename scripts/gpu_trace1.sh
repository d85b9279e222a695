for d in 0 4; do RTN_TRACE=3 RTN_DEBUG=$d python scripts/trace_tput.py 409600; done > gpurun_out/trace_tput.txt 2>&1
cat gpurun_out/trace_tput.txt
