# Epilogue cost isolation at the cfg5 shape + DSMEM store microbenchmark.
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dsmem_bench scripts/dsmem_bench.cu && /tmp/dsmem_bench > gpurun_out/dsmem.txt 2>&1
for d in 0 4 8 128; do RTN_DEBUG=$d python scripts/pair_isolate.py 409600; done > gpurun_out/isolate.txt 2>&1
for d in 0 128; do PREC=1 RTN_DEBUG=$d python scripts/pair_isolate.py 102400; done >> gpurun_out/isolate.txt 2>&1
cat gpurun_out/dsmem.txt gpurun_out/isolate.txt
