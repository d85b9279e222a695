L=5 KS=1,9,1184,2001,4736,81920 timeout 120 python scripts/ping_smoke.py; echo rc=$?
for pp in 0 1 0 1; do echo "RTN_PINGPONG=$pp"; RTN_PINGPONG=$pp timeout 200 python scripts/perf_probe.py 0 2>&1 | grep -E "256x5"; done
