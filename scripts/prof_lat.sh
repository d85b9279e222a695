set -e
mkdir -p gpurun_out
python scripts/ncu_target.py 512 12 silu 20 4 > gpurun_out/plain_lat.log 2>&1
ncu --set full --clock-control none --cache-control none --import-source on -k regex:rtn_pair -s 3 -c 1 -o gpurun_out/prof_lat_warm -f python scripts/ncu_target.py 512 12 silu 20 4 > gpurun_out/ncu_lat.log 2>&1
