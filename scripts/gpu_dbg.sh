for d in 0 4; do echo "RTN_DEBUG=$d"; RTN_KERNEL=pair RTN_DEBUG=$d timeout 100 python - <<'PY'
import sys; sys.argv=['x']; sys.path.insert(0,'scripts'); sys.path.insert(0,'.')
import perf_probe as pp
pp.probe([17]+[512]*12+[6],'silu',409600,reps=3)
pp.probe([17]+[256]*5+[6],'silu',81920,reps=3)
PY
done
mkdir -p gpurun_out
RTN_KERNEL=pair python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/plain.log 2>&1 && RTN_KERNEL=pair ncu --set full --clock-control none --import-source on -k regex:rtn_pair -s 1 -c 1 -o gpurun_out/prof_pair5 -f python scripts/ncu_target.py 512 12 silu 102400 2 > gpurun_out/ncu_pair5.log 2>&1
