"""Closed-loop errors on a conditioned 12x512 net (hidden weights x gain)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import test_gpu_closedloop as T
import oracle
from paper_2203_07747_b200 import _lib
for gain in (2.0, 2.5):
    p, cfg, om = T._setup([17] + [512] * 12 + [6], 1)
    for l, (w, b) in enumerate(om.layers()):
        if l < 12:
            om.set_layer(l, w * gain, b)
    ref = oracle.closed_loop(om, p.flat(), cfg.flat(), 20, 1, duration=0.5)
    z = np.concatenate([ref["states"][:20], np.full((20, 4), 1.84)], axis=1)
    f, j, _ = om.batched_eval(z, 1)
    print("gain", gain, "failed", ref["failed"], "ok", ref["ok"].sum(), "|f| max", np.abs(f).max(), "|J| max", np.abs(j).max())
    for prec in ("tf32", "3xtf32", "bf16x3"):
        dev = oracle.closed_loop(None, p.flat(), cfg.flat(), 20, 1, duration=0.5, prepare=T._device_prepare(om, _lib.PRECISIONS[prec]))
        print(f"  {prec:7s} state err {T._traj_err(dev['states'], ref['states']):.2e} cmd err {T._traj_err(dev['commands'], ref['commands']):.2e} failed {dev['failed']}")
