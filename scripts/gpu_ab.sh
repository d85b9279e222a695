for r in 1 2; do
for lib in paper_2203_07747_b200/librtn_mpc_prev.so paper_2203_07747_b200/librtn_mpc.so; do echo $lib; RTN_LIB=$lib timeout 200 python scripts/perf_probe.py 0 2>&1 | grep -E "K=409600|K=81920"; done
done
