for d in 0 8; do echo "RTN_DEBUG=$d"; RTN_KERNEL=pair RTN_DEBUG=$d timeout 100 python - <<'PY'
import sys; sys.argv=['x']; sys.path.insert(0,'scripts'); sys.path.insert(0,'.')
import perf_probe as pp
pp.probe([17]+[512]*12+[6],'silu',409600,reps=3)
pp.probe([17]+[256]*5+[6],'silu',81920,reps=3)
PY
done
