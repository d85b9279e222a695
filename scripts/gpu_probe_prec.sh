set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python scripts/precision_probe.py > gpurun_out/prec_o1.txt 2>&1
ORDER=2 KERNS=pair python scripts/precision_probe.py > gpurun_out/prec_o2.txt 2>&1
MEAN_SHIFT=20 PRECS=tf32,3xtf32 KERNS=pair,quad,rows python scripts/precision_probe.py > gpurun_out/prec_shift.txt 2>&1
tail -3 gpurun_out/prec_*.txt
