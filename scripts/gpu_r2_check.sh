# Round-2 kernel changes: smoke, precision per mode/kernel (orders 1, 2, generic order 2), GPU tests.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
python scripts/precision_probe.py > gpurun_out/prec_o1.txt 2>&1
ORDER=2 KERNS=pair python scripts/precision_probe.py > gpurun_out/prec_o2.txt 2>&1
GENERIC2=1 python scripts/precision_probe.py > gpurun_out/prec_g2.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
tail -n 3 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt
