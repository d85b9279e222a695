"""Prints closed-loop trajectory errors (device vs oracle) per precision mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import test_gpu_closedloop as T
import oracle
from paper_2203_07747_b200 import _lib
for sizes, order in (([17] + [512] * 12 + [6], 1), ([17, 128, 128, 128, 6], 2)):
    p, cfg, om = T._setup(sizes, order)
    ref = oracle.closed_loop(om, p.flat(), cfg.flat(), 20, order, duration=0.5)
    for prec in ("tf32", "3xtf32", "bf16x3"):
        dev = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, order, duration=0.5, prepare=T._device_prepare(om, _lib.PRECISIONS[prec]))
        fused = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, order, duration=0.5, blocks=T._device_cycle(om, p, cfg, _lib.PRECISIONS[prec]))
        print(f"{len(sizes)-2}x{sizes[1]} order {order} {prec:7s} steps {len(ref['states'])} state err prepare {T._traj_err(dev['states'], ref['states']):.2e} fused {T._traj_err(fused['states'], ref['states']):.2e} cmd err {T._traj_err(dev['commands'], ref['commands']):.2e}")
