# A/B of the blocks kernel's __launch_bounds__ min-blocks (2, 3, 4 = current, 6) on one box.
for lib in librtn_mpc_b2.so librtn_mpc_b3.so librtn_mpc.so librtn_mpc_b6.so; do
  echo "== $lib"; RTN_LIB=paper_2203_07747_b200/$lib timeout 200 python scripts/blocks_probe.py 2>&1 | grep -E '"value"|ms_per_step' | head -2
done
