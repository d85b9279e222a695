for d in 0 256 512 768; do echo "dbg $d"; RTN_DEBUG=$d timeout 60 python scripts/perf_probe.py 2>&1 | sed -n 2,2p; done
