for d in 0 16 32 48; do echo "dbg $d"; RTN_DEBUG=$d timeout 60 python scripts/trace_rows.py 2>&1 | tail -7 | head -2; done
