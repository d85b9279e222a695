for lib in minb2 minb4; do echo $lib; RTN_LIB=paper_2203_07747_b200/librtn_mpc_$lib.so NI=65536 REPS=2 timeout 120 python scripts/ncu_blocks.py; done
RTN_LIB=paper_2203_07747_b200/librtn_mpc_minb4.so timeout 300 python -m pytest tests/test_gpu_blocks.py -x -q 2>&1 | tail -3
