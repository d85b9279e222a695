# GPU test suite + smoke (round 2).
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/pytest_gpu.txt 2>&1
tail -n 25 gpurun_out/smoke.txt gpurun_out/pytest_gpu.txt
