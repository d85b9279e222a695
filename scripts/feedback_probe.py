"""Feedback-solve throughput probe: device (rtn_solve_feedback, incl. H2D/D2H) vs oracle (1 core)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle
import test_gpu_feedback as T
for n_inst, n in ((4096, 20), (4096, 50)):
    cfg, qpd, qd, xm, xs, us, om = T._setup(n_inst, n, seed=1)
    b = T._builder(om)
    b.solve_feedback(cfg, qpd, xm, xs, us)
    t0 = time.perf_counter(); r = b.solve_feedback(cfg, qpd, xm, xs, us); t = time.perf_counter() - t0
    ns = 64
    t1 = time.perf_counter(); oracle.solve_feedback(n, {k: v[:ns] for k, v in qd.items() if k != "f_evals"}, xm[:ns], xs[:ns], us[:ns]); tc = time.perf_counter() - t1
    print(f"N={n} n_inst={n_inst}: device {n_inst / t:.0f} inst/s ({t*1e3:.1f} ms, iters mean {r.iterations.mean():.1f}), "
          f"oracle 1 core {ns / tc:.0f} inst/s")
