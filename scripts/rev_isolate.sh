for d in 0 2 4 6; do
RTN_DEBUG=$d JMODE=1 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/rev_d$d.csv timeout 300 python scripts/pair_isolate.py 131072 > /dev/null 2>&1
done
