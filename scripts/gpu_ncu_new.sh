CFG=cfg3 timeout 60 python scripts/ncu_small.py && CFG=cfg4 timeout 60 python scripts/ncu_small.py || exit 1
CFG=cfg3 REPS=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:rtn_quad_kernel -s 2 -c 1 -o gpurun_out/ncu_quad -f python scripts/ncu_small.py > gpurun_out/ncu_quad.log 2>&1; tail -1 gpurun_out/ncu_quad.log
CFG=cfg4 REPS=3 timeout 600 ncu --set full --import-source on --clock-control none -k regex:rtn_pingpong_kernel -s 2 -c 1 -o gpurun_out/ncu_ping -f python scripts/ncu_small.py > gpurun_out/ncu_ping.log 2>&1; tail -1 gpurun_out/ncu_ping.log
