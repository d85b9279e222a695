# Round-2 ncu captures of the kernels added late in the round: the BF16 rowsb
# kernel and the two reverse-mode passes (cfg5 shape, one launch each).
set -x
mkdir -p gpurun_out
python scripts/ncu_target.py 512 12 silu 102400 2 bf16 > gpurun_out/plainb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:rtn_rowsb -s 1 -c 1 -o gpurun_out/prof_r02_rowsb -f \
    python scripts/ncu_target.py 512 12 silu 102400 2 bf16 > gpurun_out/ncu_rowsb.log 2>&1
JMODE=1 python scripts/pair_isolate.py 65536 > gpurun_out/plainr.log 2>&1 && \
JMODE=1 ncu --set full --clock-control none --import-source on -k regex:rtn_rev -s 2 -c 2 -o gpurun_out/prof_r02_rev -f \
    python scripts/pair_isolate.py 65536 > gpurun_out/ncu_rev.log 2>&1
ls -la gpurun_out | tail -4
