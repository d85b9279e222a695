for r in 1 2; do for lib in reg ce; do echo $lib; RTN_LIB=paper_2203_07747_b200/librtn_mpc_$lib.so timeout 200 python scripts/perf_probe.py 0 2>&1 | grep -E "K=409600"; done; done
timeout 600 python -m pytest tests/test_gpu_blocks.py tests/test_gpu_parity.py -q 2>&1 | tail -1
