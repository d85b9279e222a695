# same-box A/B of the rows kernel (cfg4 line of perf_probe): previous build vs current, twice
for r in 1 2; do
for lib in paper_2203_07747_b200/librtn_mpc_prev.so paper_2203_07747_b200/librtn_mpc.so; do
  echo "$lib"; RTN_LIB=$lib timeout 120 python scripts/perf_probe.py 0 2>&1 | grep "K=81920"
done
done
RTN_KERNEL=rows timeout 90 python -m pytest tests/test_gpu_parity.py -q -x -k "rows" 2>&1 | tail -1
