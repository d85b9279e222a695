ORDER=1 timeout 120 python scripts/cycle_probe.py
ORDER=2 timeout 120 python scripts/cycle_probe.py
ORDER=1 REPS=20 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cycle1_launches.csv python scripts/cycle_probe.py > /dev/null 2>&1
ORDER=2 REPS=20 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cycle2_launches.csv python scripts/cycle_probe.py > /dev/null 2>&1
tail -4 gpurun_out/cycle1_launches.csv; tail -4 gpurun_out/cycle2_launches.csv
