"""Benchmark: node linearisations/s of (f, ∂f/∂x, ∂f/∂u) on the BASELINE
workload, plus p50/p99 per-MPC-step latency, roofline and CPU baseline.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL). Workload (N=1 and
every N, strong scaling): BASELINE.json configs[4] — 65,536 MPC instances x
N=50 shooting nodes, quadrotor residual MLP 12x512 SiLU (17 in, 6 out),
first order, TF32 tensor cores; instances are partitioned across ranks and
the (f, A, B) blocks are gathered to rank 0 with NCCL (the path's only
exchange step). Synthetic inputs: MakeMlp weights (seed 12512) and
quadrotor node rows (mt19937_64), inputs resident in HBM.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "node linearizations/s (f,∂f/∂x,∂f/∂u) at 1-8 GPU; p50 per-MPC-step latency"
UNIT = "node-lin/s"
INSTANCES, HORIZON = 65536, 50
SIZES = [17] + [512] * 12 + [6]
SEED = 1000 * 12 + 512
WORKLOAD = "cfg5: 65536 MPC instances x N=50 nodes, quadrotor MLP 12x512 SiLU (17->6), order 1"


def _env_int(k, d):
    try:
        return int(os.environ.get(k, d))
    except ValueError:
        return d


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-f", self.path], stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        try:
            rows = [r.split(",") for r in open(self.path).read().strip().splitlines() if r.strip()]
        except Exception:
            rows = []
        finally:
            if self.path and os.path.exists(self.path):
                os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].strip().replace(".", "").isdigit()]
        smax = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if "Active" in v and "Not" not in v})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": reasons,
                "samples": len(rows)}


# --------------------------------------------------------------------------- CPU (oracle) leg
def cpu_throughput(target_s: float, threads: int, sizes=SIZES, seed=SEED):
    """The reference's CPU algorithm (oracle/ restatement of BatchedCore,
    reverse-mode fp64, RESMPC thread pool) on a bounded sample of the same
    workload; sample size calibrated to ~target_s seconds."""
    import numpy as np
    import oracle
    om = oracle.OracleModel.make_mlp(sizes, "silu", seed)
    z = oracle.quad_nodes(2203, 50 * 64)
    t0 = time.perf_counter()
    om.batched_eval(z[:HORIZON * 2], 1, threads)  # calibration: 2 instances
    dt = max(time.perf_counter() - t0, 1e-4)
    per_node = dt / (HORIZON * 2)
    inst = int(max(1, min(64, target_s / (per_node * HORIZON))))
    k = inst * HORIZON
    t0 = time.perf_counter()
    om.batched_eval(z[:k], 1, threads)
    dt = time.perf_counter() - t0
    return k / dt, f"{inst} instances x {HORIZON} nodes = {k} nodes of cfg5 in {dt:.2f} s", dt


def run_reference(args, rank, world):
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    per_step = max(1.0, min(20.0, 150.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        cpu_throughput(per_step, threads)
    vals, samples = [], []
    for _ in range(args.steps):
        v, sample, _ = cpu_throughput(per_step, threads)
        vals.append(v)
        samples.append(sample)
    v = statistics.median(vals)
    line = {
        "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * INSTANCES * HORIZON / v, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": WORKLOAD, "nodes": INSTANCES * HORIZON,
                   "note": "reference algorithm = oracle/ restatement of proj/src/neural.cpp BatchedCore "
                           "(reverse mode, fp64, fork/join pool); the reference itself needs Eigen/yaml-cpp "
                           "and cannot be built here; ms_per_step extrapolated linearly from the sample"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": threads, "kind": "port", "sample": samples[-1]},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU leg
def measured_tf32_peak(torch):
    """cuBLAS TF32 8192^3 burst on this GPU (the tensor-core roofline the
    kernel is compared against); MEASURED_PEAKS.json only carries bf16."""
    torch.backends.cuda.matmul.allow_tf32 = True
    a = torch.randn(8192, 8192, device="cuda")
    b = torch.randn(8192, 8192, device="cuda")
    for _ in range(3):
        a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        a @ b
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2 * 8192 ** 3 / (best * 1e-3) / 1e12


def latency(torch, sizes, seed, k, steps=1000, warm=50, order=1, precision=0):
    """Per-MPC-step approximation latency: K = N nodes of one instance
    through rtn_prepare (host z -> host f, J), and device-only (events)."""
    import numpy as np
    from paper_2203_07747_b200 import _lib, make_mlp, synth_quad_nodes
    from paper_2203_07747_b200.errors import raise_for_status
    m = make_mlp(sizes, "silu", "full", seed)
    eng = m.engine(latency_mode=1, precision=precision)  # graph-captured H2D -> kernel -> D2H per step
    eng._ensure(k, order)
    L = _lib.lib()
    z = torch.from_numpy(synth_quad_nodes(7, k)).pin_memory()
    f = torch.empty((k, sizes[-1]), dtype=torch.float64).pin_memory()
    j = torch.empty((k, sizes[-1], sizes[0]), dtype=torch.float64).pin_memory()
    h = torch.empty((k, sizes[-1], sizes[0], sizes[0]), dtype=torch.float64).pin_memory() if order == 2 else None
    dp = C.POINTER(C.c_double)
    args = (eng.ctx_ptr, C.cast(z.data_ptr(), dp), k, sizes[0], order, C.cast(f.data_ptr(), dp), C.cast(j.data_ptr(), dp),
            C.cast(h.data_ptr(), dp) if h is not None else None)
    for _ in range(warm):
        raise_for_status(L.rtn_prepare(*args))
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        L.rtn_prepare(*args)
        ts.append((time.perf_counter() - t0) * 1e6)
    # device-only: kernel on device-resident rows
    st = torch.cuda.Stream()
    raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
    dz = z.cuda()
    df = torch.empty((k, sizes[-1]), dtype=torch.float64, device="cuda")
    dj = torch.empty((k, sizes[-1], sizes[0]), dtype=torch.float64, device="cuda")
    dh = torch.empty((k, sizes[-1], sizes[0], sizes[0]), dtype=torch.float64, device="cuda") if order == 2 else None
    dev = []
    with torch.cuda.stream(st):
        for i in range(warm + 200):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            L.rtn_prepare_device(eng.ctx_ptr, dz.data_ptr(), k, order, df.data_ptr(), dj.data_ptr(),
                                 dh.data_ptr() if dh is not None else None)
            e1.record(st)
            e1.synchronize()
            if i >= warm:
                dev.append(e0.elapsed_time(e1) * 1e3)
    raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, None))
    ts.sort()
    dev.sort()
    return {"p50_us": ts[len(ts) // 2], "p99_us": ts[int(len(ts) * 0.99)], "device_p50_us": dev[len(dev) // 2],
            "device_p99_us": dev[int(len(dev) * 0.99)], "steps": steps}


def precision_modes(torch, z, k, sizes, steps=2):
    """Same workload in the split-precision modes (device-resident, 1 warm-up
    + `steps` timed launches each). Accuracy per mode is pinned by
    tests/test_gpu_precision.py."""
    from paper_2203_07747_b200 import _lib, flops_per_node, make_mlp
    from paper_2203_07747_b200.errors import raise_for_status
    L = _lib.lib()
    out = {}
    fl = flops_per_node(sizes, 1)
    for name in ("bf16x3", "3xtf32"):
        m = make_mlp(sizes, "silu", "full", SEED)
        eng = m.engine(precision=_lib.PRECISIONS[name])
        eng._ensure(k, 1)
        st = torch.cuda.Stream()
        raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
        f = torch.empty((k, sizes[-1]), dtype=torch.float64, device="cuda")
        j = torch.empty((k, sizes[-1], sizes[0]), dtype=torch.float64, device="cuda")
        run = lambda: raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(), j.data_ptr(), None))
        with torch.cuda.stream(st):
            run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(steps):
                run()
            e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out[name] = {"value": k / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "achieved_tflops": k * fl / (ms * 1e-3) / 1e12}
        eng.close()
        del f, j
    return out


def cfg4_bench(torch, tf32_peak, steps=5):
    """BASELINE configs[3]: 4096 instances x N=20 x MLP 5x256 SiLU, throughput mode on
    1 B200, TF32 and 3xTF32 (device-resident, CUDA events on the launching stream)."""
    from paper_2203_07747_b200 import _lib, flops_per_node, make_mlp, synth_quad_nodes
    from paper_2203_07747_b200.errors import raise_for_status
    L = _lib.lib()
    sizes, k = [17] + [256] * 5 + [6], 4096 * 20
    fl = flops_per_node(sizes, 1)
    z = torch.from_numpy(synth_quad_nodes(2203, k)).cuda()
    f = torch.empty((k, 6), dtype=torch.float64, device="cuda")
    j = torch.empty((k, 6, 17), dtype=torch.float64, device="cuda")
    out = {"workload": "cfg4: 4096 instances x N=20 nodes, MLP 5x256 SiLU (17->6), order 1", "nodes": k}
    for name in ("tf32", "3xtf32"):
        m = make_mlp(sizes, "silu", "full", 5256)
        eng = m.engine(precision=_lib.PRECISIONS[name])
        eng._ensure(k, 1)
        st = torch.cuda.Stream()
        raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
        run = lambda: raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(),
                                                            j.data_ptr(), None))
        with torch.cuda.stream(st):
            for _ in range(3):
                run()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(steps):
                run()
            e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        ach = k * fl / (ms * 1e-3) / 1e12
        out[name] = {"value": k / (ms * 1e-3), "unit": UNIT, "ms_per_step": ms, "achieved_tflops": ach,
                     "kernel": ("rtn_rows_kernel (activations as the A operand in TMEM, M = 256 rows x N = 256)"
                                if name == "tf32" else "rtn_pair_kernel<256,4,4,80,3xTF32> (split accumulators)"),
                     "frac_of_tf32_peak": ach / tf32_peak if tf32_peak else None,
                     "hardware_frac": (3 if name == "3xtf32" else 1) * ach / tf32_peak if tf32_peak else None}
        eng.close()
    return out


def feedback_bench():
    """§8f rank 4: the batched feedback solve (csrc/rtn_qpsolve.cu: condensing + primal
    active-set box QP + recovery, fp64) through rtn_solve_feedback (host buffers in and
    out). QpData come from the product's own BuildQp (rtn_build_qp) on synthetic
    quadrotor iterates and approximations; the oracle's SolveFeedback on one host core
    is timed beside it (cpu_baseline)."""
    import numpy as np
    import oracle
    from paper_2203_07747_b200 import make_mlp, qp
    out = {}
    for n_inst, n in ((4096, 20), (1024, 50)):
        xs, us, rx, ru = _quad_iterate(np, n_inst, n, 1)
        rng = np.random.default_rng(2)
        k = n_inst * n
        z0 = np.concatenate([xs[:, :n], us], axis=-1).reshape(k, 17)
        fb, jac = rng.normal(0, 0.5, (k, 6)), rng.normal(0, 0.1, (k, 6, 17))
        xm = xs[:, 0, :] + rng.normal(0, 0.1, (n_inst, 13))
        cfg = qp.OcpConfig(horizon=n, dt=0.05, q_diag=np.array([10, 10, 10, 1, 1, 1, 1, 1, 1, 1, .1, .1, .1]),
                           r_diag=np.full(4, 0.1), u_min=np.zeros(4), u_max=np.full(4, 6.0))
        b = qp.QpBuilder(make_mlp([17, 64, 6], "silu", "full", 1))
        qpd = b.build_qp(qp.QuadParams(), cfg, xs, us, rx, ru, {"z0": z0, "f_bar": fb, "jac": jac})
        b.solve_feedback(cfg, qpd, xm, xs, us)
        t0 = time.perf_counter()
        r = b.solve_feedback(cfg, qpd, xm, xs, us)
        t = time.perf_counter() - t0
        ns = 32
        sub = {f: getattr(qpd, f)[:ns] for f in ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag", "du_lb", "du_ub")}
        t1 = time.perf_counter()
        oracle.solve_feedback(n, sub, xm[:ns], xs[:ns], us[:ns])
        tc = time.perf_counter() - t1
        out[f"N{n}"] = {"value": n_inst / t, "unit": "instances/s", "instances": n_inst, "ms": t * 1e3,
                        "optimal": int((r.status == 0).sum()),
                        "mean_active_set_passes": float(r.iterations.mean()),
                        "path": "rtn_solve_feedback (C-ABI), host QpData in, steps/commands out",
                        "cpu_baseline": {"value": ns / tc, "unit": "instances/s", "cores": 1, "kind": "port",
                                         "sample": f"{ns} instances in {tc:.2f} s"}}
        b.engine.close()
    return out


def _quad_iterate(np, n_inst, n, seed):
    rng = np.random.default_rng(seed)
    xs = np.empty((n_inst, n + 1, 13))
    xs[..., 0:3] = rng.uniform(-2, 2, (n_inst, n + 1, 3))
    q = rng.uniform(-1, 1, (n_inst, n + 1, 4))
    xs[..., 3:7] = q / np.linalg.norm(q, axis=-1, keepdims=True)
    xs[..., 7:10] = rng.uniform(-4, 4, (n_inst, n + 1, 3))
    xs[..., 10:13] = rng.uniform(-3, 3, (n_inst, n + 1, 3))
    us = rng.uniform(0.5, 5.0, (n_inst, n, 4))
    return xs, us, xs + rng.normal(0, 0.1, xs.shape), us + rng.normal(0, 0.1, us.shape)


def blocks_bench(torch, hbm_peak, steps=5):
    """§8f rank 1: the continuity-block builder (csrc/rtn_blocks.cu) on the
    cfg5 shape (65,536 instances x N=50), fp64. Device-resident throughput
    with the HBM roofline, e2e through rtn_build_qp (pinned host buffers),
    the fused PrepareNodes+BuildQp cycle latency at cfg3, and the oracle
    BuildQp on the host as the CPU baseline."""
    import numpy as np
    import oracle
    from paper_2203_07747_b200 import _lib, make_mlp, qp
    from paper_2203_07747_b200.errors import raise_for_status
    L = _lib.lib()
    n_inst, n = INSTANCES, HORIZON
    k = n_inst * n
    xs, us, rx, ru = _quad_iterate(np, n_inst, n, 2203)
    rng = np.random.default_rng(5)
    z0 = np.concatenate([xs[:, :n], us], axis=-1).reshape(k, 17)
    fb = rng.normal(0, 0.5, (k, 6))
    jac = rng.normal(0, 0.1, (k, 6, 17))
    p, cfg = qp.QuadParams(), qp.OcpConfig(horizon=n, dt=0.02, q_diag=np.ones(13), r_diag=np.full(4, 0.1))
    model = make_mlp([17, 64, 6], "silu", "full", 1)  # context owner only; the builder does not touch it
    eng = model.engine()
    eng._ensure(k, 1)
    st = torch.cuda.Stream()
    raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(st.cuda_stream)))
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    d_in = [dev(a) for a in (xs, us, rx, ru, z0, fb, jac)]
    shapes = {"a": (k, 13, 13), "b": (k, 13, 4), "phi_res": (k, 13), "q": (n_inst, n + 1, 13), "r": (k, 4),
              "hx_diag": (n_inst, n + 1, 13), "hu_diag": (k, 4), "du_lb": (k, 4), "du_ub": (k, 4)}
    d_out = {name: torch.empty(s, dtype=torch.float64, device="cuda") for name, s in shapes.items()}
    it = _lib.IterateC(*[t.data_ptr() for t in d_in[:4]])
    ap = _lib.ApproxC(d_in[4].data_ptr(), d_in[5].data_ptr(), d_in[6].data_ptr(), None)
    oc = _lib.QpBlocksC(*[d_out[nm].data_ptr() for nm in ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag",
                                                             "du_lb", "du_ub")])
    pc, cc = p.to_c(), cfg.to_c()
    run = lambda: raise_for_status(L.rtn_build_qp_device(eng.ctx_ptr, C.byref(pc), C.byref(cc), n_inst, C.byref(it),
                                                         C.byref(ap), C.byref(oc)))
    with torch.cuda.stream(st):
        run()
        ms = []
        for _ in range(steps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            run()
            e1.record(st)
            e1.synchronize()
            ms.append(e0.elapsed_time(e1))
    t = statistics.median(ms)
    in_b = sum(a.numel() for a in d_in) * 8
    out_b = sum(v.numel() for v in d_out.values()) * 8
    gbs = (in_b + out_b) / (t * 1e-3) / 1e9
    raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, None))
    # e2e: the C-ABI call a user makes, pinned host buffers in and out
    h_in = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in (xs, us, rx, ru, z0, fb, jac)]
    h_out = {name: torch.empty(s, dtype=torch.float64).pin_memory() for name, s in shapes.items()}
    hit = _lib.IterateC(*[t_.data_ptr() for t_ in h_in[:4]])
    hap = _lib.ApproxC(h_in[4].data_ptr(), h_in[5].data_ptr(), h_in[6].data_ptr(), None)
    hoc = _lib.QpBlocksC(*[h_out[nm].data_ptr() for nm in ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag",
                                                              "du_lb", "du_ub")])
    hrun = lambda: raise_for_status(L.rtn_build_qp(eng.ctx_ptr, C.byref(pc), C.byref(cc), n_inst, C.byref(hit),
                                                   C.byref(hap), C.byref(hoc), None))
    hrun()
    t0 = time.perf_counter()
    for _ in range(2):
        hrun()
    e2e_s = (time.perf_counter() - t0) / 2
    same = bool(torch.equal(h_out["a"], d_out["a"].cpu()))
    del d_in, d_out, h_in, h_out
    eng.close()
    # fused phase 1+2 latency at cfg3 (12x512, N=20, one instance), host -> host through the
    # C-ABI (rtn_cycle_qp, structs built once like a controller would), and device-only
    lat = {}
    big = make_mlp(SIZES, "silu", "full", SEED)
    for order in (1, 2):
        b = qp.QpBuilder(big, latency_mode=1)
        b.engine._ensure(20, order)
        cfg3 = qp.OcpConfig(horizon=20, dt=0.02, q_diag=np.ones(13), r_diag=np.full(4, 0.1), taylor_order=order)
        x3, u3, rx3, ru3 = (np.ascontiguousarray(a[0]) for a in _quad_iterate(np, 1, 20, 3))
        outs = {nm: np.empty(sh) for nm, sh in {"a": (20, 13, 13), "b": (20, 13, 4), "phi_res": (20, 13),
                                                 "q": (21, 13), "r": (20, 4), "hx_diag": (21, 13), "hu_diag": (20, 4),
                                                 "du_lb": (20, 4), "du_ub": (20, 4)}.items()}
        it3 = _lib.IterateC(x3.ctypes.data, u3.ctypes.data, rx3.ctypes.data, ru3.ctypes.data)
        oc3 = _lib.QpBlocksC(*[outs[nm].ctypes.data for nm in ("a", "b", "phi_res", "q", "r", "hx_diag", "hu_diag",
                                                                "du_lb", "du_ub")])
        pc3, cc3 = p.to_c(), cfg3.to_c()
        args = (b.engine.ctx_ptr, C.byref(pc3), C.byref(cc3), 1, C.byref(it3), C.byref(oc3), None, None, None)
        for _ in range(50):
            raise_for_status(L.rtn_cycle_qp(*args))
        ts = []
        for _ in range(300 if order == 2 else 1000):
            t0 = time.perf_counter()
            L.rtn_cycle_qp(*args)
            ts.append((time.perf_counter() - t0) * 1e6)
        ts.sort()
        lat[f"cfg3_cycle_order{order}"] = {"p50_us": ts[len(ts) // 2], "p99_us": ts[int(len(ts) * 0.99)],
                                           "steps": len(ts),
                                           "path": "rtn_cycle_qp (C-ABI): H2D iterate -> [x;u] features -> MLP (f,A,B" +
                                                   (",H" if order == 2 else "") + ") -> RK4 blocks -> D2H QpData, "
                                                   "one CUDA graph"}
    big.invalidate()
    # CPU baseline: the oracle's serial BuildQp (like the reference's per-instance loop)
    ns = 64
    t0 = time.perf_counter()
    oracle.build_qp_quad(p.flat(), cfg.flat(), n, 0, 1, xs[:ns], us[:ns], rx[:ns], ru[:ns], z0[:ns * n], fb[:ns * n],
                         jac[:ns * n])
    cpu_s = time.perf_counter() - t0
    return {"metric": "continuity blocks/s (A 13x13, B 13x4, phi_res + cost terms per node, fp64)",
            "value": k / (t * 1e-3), "unit": "node-blocks/s", "ms_per_step": t, "nodes": k,
            "kernel": "QpBlocksKernel (warp per node, fp64)", "gpu_launches_per_step": 1,
            "roofline": {"bound": "hbm", "achieved": gbs, "peak": hbm_peak, "unit": "GB/s",
                         "frac": gbs / hbm_peak if hbm_peak else None, "bytes_per_node": (in_b + out_b) / k,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs"},
            "e2e": {"value": k / e2e_s, "unit": "node-blocks/s", "h2d_bytes_per_step": in_b, "d2h_bytes_per_step": out_b,
                    "path": "rtn_build_qp (C-ABI), pinned host buffers", "matches_device_run": same},
            "cpu_baseline": {"value": ns * n / cpu_s, "unit": "node-blocks/s", "cores": 1, "kind": "port",
                             "sample": f"{ns} instances x {n} nodes in {cpu_s:.2f} s",
                             "algorithm": "oracle/blocks_oracle.cpp BuildQp (sqp_rti.cpp:59-155), serial like the reference"},
            "latency": lat}


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2203_07747_b200 import _lib, flops_per_node, make_mlp, synth_quad_nodes
    from paper_2203_07747_b200.errors import raise_for_status
    from paper_2203_07747_b200.sharding import partition_instances

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    part = partition_instances(INSTANCES, HORIZON, rank, world)
    k = part.num_nodes
    n_in, n_out = SIZES[0], SIZES[-1]
    L = _lib.lib()

    tf32_peak = measured_tf32_peak(torch) if rank == 0 else None

    model = make_mlp(SIZES, "silu", "full", SEED)
    eng = model.engine(device=local_rank)
    eng._ensure(k, 1)
    stream = torch.cuda.Stream(device=dev)
    raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, C.c_void_p(stream.cuda_stream)))

    z_host = torch.from_numpy(synth_quad_nodes(2203 + rank, k))
    z = z_host.to(dev)
    # kernel outputs are the gather send buffers (no extra copy in the step)
    f = torch.empty((k, n_out), dtype=torch.float64, device=dev)
    jac = torch.empty((k, n_out, n_in), dtype=torch.float64, device=dev)
    k_max = partition_instances(INSTANCES, HORIZON, 0, world).num_nodes
    if world > 1:
        f_send = torch.zeros((k_max, n_out), dtype=torch.float64, device=dev)
        j_send = torch.zeros((k_max, n_out, n_in), dtype=torch.float64, device=dev)
        f, jac = f_send[:k], j_send[:k]
        f_recv = [torch.empty_like(f_send) for _ in range(world)] if rank == 0 else None
        j_recv = [torch.empty_like(j_send) for _ in range(world)] if rank == 0 else None

    def launches():
        a, b, c = C.c_ulonglong(), C.c_ulonglong(), C.c_ulonglong()
        L.rtn_ctx_counters(eng.ctx_ptr, C.byref(a), C.byref(b), C.byref(c))
        return c.value

    kern_ms = []

    def step(record_kernel):
        e0 = e1 = None
        with torch.cuda.stream(stream):
            if record_kernel:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
            raise_for_status(L.rtn_prepare_device(eng.ctx_ptr, z.data_ptr(), k, 1, f.data_ptr(), jac.data_ptr(), None))
            if record_kernel:
                e1.record(stream)
            if world > 1:
                dist.gather(f_send, f_recv, dst=0)
                dist.gather(j_send, j_recv, dst=0)
        return (e0, e1)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local_rank])
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        step(False)
    barrier()
    l0 = launches()
    ev_pairs = []
    with ClockSampler(local_rank) as clk:
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0.record(stream)
        for _ in range(args.steps):
            ev_pairs.append(step(True))
        t1.record(stream)
        barrier()
    clocks = clk.summary()
    n_launch = launches() - l0
    elapsed = t0.elapsed_time(t1)
    kern_ms = [a.elapsed_time(b) for a, b in ev_pairs]
    tmax = torch.tensor([elapsed], dtype=torch.float64, device=dev)
    kmax = torch.tensor([statistics.mean(kern_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(kmax, op=dist.ReduceOp.MAX)
    ms_per_step = float(tmax.item()) / args.steps
    kernel_ms = float(kmax.item())
    total_nodes = INSTANCES * HORIZON
    value = total_nodes / (ms_per_step * 1e-3)

    # ---- end to end through the public C-ABI: pinned host z -> host f, J
    zp = z_host.pin_memory()
    fp = torch.empty((k, n_out), dtype=torch.float64).pin_memory()
    jp = torch.empty((k, n_out, n_in), dtype=torch.float64).pin_memory()
    dp = C.POINTER(C.c_double)
    e2e_args = (eng.ctx_ptr, C.cast(zp.data_ptr(), dp), k, n_in, 1, C.cast(fp.data_ptr(), dp),
                C.cast(jp.data_ptr(), dp), None)
    raise_for_status(L.rtn_ctx_set_stream(eng.ctx_ptr, None))
    raise_for_status(L.rtn_prepare(*e2e_args))  # warm
    barrier()
    e2e_steps = max(1, min(args.steps, 3))
    t_e2e = time.perf_counter()
    for _ in range(e2e_steps):
        raise_for_status(L.rtn_prepare(*e2e_args))
    e2e_s = torch.tensor([(time.perf_counter() - t_e2e) / e2e_steps], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = total_nodes / float(e2e_s.item())
    # sanity: outputs finite and match the device-resident run
    ok = bool(torch.isfinite(fp).all()) and bool(torch.allclose(fp, f.cpu(), rtol=0, atol=0))

    result = None
    if rank == 0:
        fl = flops_per_node(SIZES, 1)
        achieved = k * fl / (kernel_ms * 1e-3) / 1e12
        peaks = {}
        try:
            peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        except Exception:
            pass
        traffic = None
        try:
            prof = json.load(open(os.path.join(ROOT, "profiles", "roofline_traffic.json")))
            traffic = prof.get("dram_bytes_per_launch_per_node", None)
            traffic = traffic * k if traffic is not None else None
        except Exception:
            pass
        cpu = None
        if world == 1 and not args.no_cpu:
            threads = os.cpu_count() or 1
            v_all, sample, _ = cpu_throughput(12.0, threads)
            v_one, sample1, _ = cpu_throughput(3.0, 1)
            cpu = {"value": v_all, "unit": UNIT, "cores": threads, "kind": "port", "sample": sample,
                   "value_1thread": v_one, "sample_1thread": sample1,
                   "algorithm": "oracle/ restatement of proj/src/neural.cpp BatchedCore (reverse mode, fp64)"}
        modes = None
        if world == 1 and not args.no_modes:
            modes = precision_modes(torch, z, k, SIZES)
        lat = None
        if not args.no_latency:
            lat = {"cfg3_12x512_N20": latency(torch, SIZES, SEED, 20),
                   "cfg3_12x512_N20_order2": latency(torch, SIZES, SEED, 20, steps=300, order=2),
                   "cfg3_12x512_N20_bf16x3": latency(torch, SIZES, SEED, 20, steps=300, precision=2),
                   "cfg3_12x512_N20_3xtf32": latency(torch, SIZES, SEED, 20, steps=300, precision=1),
                   "cfg2_5x256_N20": latency(torch, [17] + [256] * 5 + [6], 5256, 20),
                   "cfg1_2x64_N10": latency(torch, [17, 64, 64, 6], 2064, 10, steps=300)}
        cfg4 = cfg4_bench(torch, tf32_peak) if world == 1 and not args.no_modes else None
        blocks = None
        if world == 1 and not args.no_blocks:
            blocks = blocks_bench(torch, peaks.get("hbm_gbs"))
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "tf32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "nodes": total_nodes, "nodes_per_rank": k,
                       "parallelism": f"instance partition x{world}" + (" + NCCL gather of (f,A,B) to rank 0" if world > 1 else ""),
                       "l2": "inputs larger than L2 (z 446 MB + outputs 2.8 GB per step); weights (11.6 MB) stay L2-resident by design",
                       "io": "fp64 z in, fp64 f/J out (reference layout)"},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(zp.numel() * 8),
                    "d2h_bytes_per_step": int((fp.numel() + jp.numel()) * 8),
                    "path": "rtn_prepare (C-ABI), pinned host buffers, chunked H2D/kernel/D2H overlap",
                    "matches_device_run": ok},
            "gpu_launches": int(n_launch),
            "kernel_ms": kernel_ms,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": tf32_peak, "unit": "TFLOP/s",
                         "frac": achieved / tf32_peak if tf32_peak else None, "traffic": traffic,
                         "peak_source": "cuBLAS tf32 8192^3 burst measured in this run (MEASURED_PEAKS.json has bf16 only; "
                                        f"bf16/2 = {peaks.get('bf16_tflops', 0) / 2:.1f})",
                         "flop_per_node": fl, "flops_definition": "2*(1+n_in)*sum(n_l*n_{l+1}) forward-mode (BASELINE.md s2)",
                         "kernel": "rtn_pair_kernel<512,4,4> (tcgen05 cta_group::2 tf32)"},
            "clocks": clocks,
        }
        if cpu:
            result["cpu_baseline"] = cpu
        if modes:
            result["precision_modes"] = modes
        if lat:
            result["latency"] = lat
        if cfg4:
            result["cfg4"] = cfg4
        if blocks:
            result["blocks"] = blocks
            result["feedback"] = feedback_bench()
    if world > 1:
        dist.barrier(device_ids=[local_rank])
        dist.destroy_process_group()
    if result is not None:
        print(json.dumps(result), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-latency", action="store_true")
    ap.add_argument("--no-modes", action="store_true")
    ap.add_argument("--no-blocks", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    rank = _env_int("RANK", 0)
    world = _env_int("WORLD_SIZE", 1)
    local_rank = _env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
