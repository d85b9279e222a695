# same-box A/B of the latency kernels (cfg3 per mode and order 2): previous build vs current
for lib in paper_2203_07747_b200/librtn_mpc_prev.so paper_2203_07747_b200/librtn_mpc.so; do
  echo "$lib"; RTN_LIB=$lib timeout 200 python scripts/lat_probe.py 2>&1 | tail -2; RTN_LIB=$lib timeout 200 python scripts/lat_modes.py 2>&1 | tail -3
done
