"""Benchmark: planned steps/sec (and curvature products/sec) of the curvopt hot path on B200.

Default workload (BASELINE.json configs[2], "C3"): MLP 784-1024-1024-10 softmax-CE,
global batch 8192, GGN curvature, PCG (tol 1e-5, maxiter 10, stabilise 10, warm
start) with the diag-EMA(0.99) preconditioner fed by a Hutchinson probe every 10
steps, constant damping lam = 1, chain (scale 1e-3, scale -1).  Synthetic data from
the reference's SplitMix64 stream (MNIST-shaped), random-init weights (init_params).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3|c4|c5]

--config c4: configs[3], row-space lane (Gram + Cholesky), 3072-2048-2048-10, b=4096.
--config c5: configs[4], exact-Hessian HVP + CG + trace/diag telemetry,
             3072-4096x4-10, b=32768 (on N GPUs: b/N rows per rank).
--config cadence: the paper's only published measurement of this path (PAPER.md
             Table 3): newton_cg on MLP 512-1024-1024-1, b=256, constant damping,
             CG maxiter 3, rho_every_k in {-1, 10, 5, 2, 1}, paired step timing
             (harness.bench_cadence); value = median step ms with rho off.

With N GPUs the global batch is sharded b/N per rank (strong scaling: the total work
is fixed); every gradient and curvature product is NCCL all-reduced inside the native
library.  Without torchrun, `--gpus N` (N > 1) launches the N ranks itself.

Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import platform
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "GGN-CG planned steps/sec (C3: 784-1024-1024-10, b=8192, PCG + diag-EMA)"
UNIT = "steps/s"


class Workload:
    def __init__(self, key, dims, b, metric, desc, kind, lane):
        self.key, self.dims, self.b, self.metric, self.desc, self.kind, self.lane = key, dims, b, metric, desc, kind, lane

    def config(self, world):
        return {"workload": self.desc, "global_batch": self.b, "dims": list(self.dims),
                "parallelism": f"dp{world}" if self.lane == "param" or world == 1 else
                f"dp{world} (row lane: Gram strips + Cholesky block-cyclic over {world} ranks)",
                "l2": "per-step working set > 126 MB L2 (no flush)"}


WORKLOADS = {
    "c3": Workload("c3", (784, 1024, 1024, 10), 8192, METRIC,
                   "C3 784-1024-1024-10 softmax-CE, GGN + PCG(diag-EMA 0.99, Hutchinson@10), lam=1, "
                   "CG tol 1e-5 maxiter 10", "ggn", "param"),
    "c4": Workload("c4", (3072, 2048, 2048, 10), 4096,
                   "row-space planned steps/sec (C4: 3072-2048-2048-10, b=4096, Gram + Cholesky)",
                   "C4 3072-2048-2048-10 softmax-CE, GGN row-space lane: Gram JJ^T + mu I (m=40960) + blocked "
                   "Cholesky + backprojection, lam=1", "ggn", "row"),
    "c5": Workload("c5", (3072, 4096, 4096, 4096, 4096, 10), 32768,
                   "exact-Hessian HVP-CG planned steps/sec (C5: 3072-4096x4-10, b=32768)",
                   "C5 3072-4096x4-10 softmax-CE, exact-Hessian HVP + CG (tol 1e-5, maxiter 10), constant lam=1 "
                   "(the reference has no step-norm damping), Hutchinson diag + trace telemetry @10", "hessian",
                   "param"),
}
DIMS = WORKLOADS["c3"].dims
GLOBAL_B = WORKLOADS["c3"].b


def P_w(dims):
    return sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))


def gv_flops(dims, b):
    """Useful fp32-equivalent flops of one GGN product: 8 b P_w - 4 b n0 n1."""
    return 8 * b * P_w(dims) - 4 * b * dims[0] * dims[1]


def hvp_flops(dims, b):
    """One exact-Hessian product (ReLU): 12 b P_w - 8 b n0 n1."""
    return 12 * b * P_w(dims) - 8 * b * dims[0] * dims[1]


def row_flops(dims, b):
    """Row lane: Gram as SYRK sum_l m^2 n_{l+1} + potrf m^3/3."""
    c = dims[-1]
    m = b * c
    return sum(m * m * dims[l + 1] for l in range(len(dims) - 1)) + m ** 3 / 3.0


def make_batches(n_batches, b_global, rank, world, dims=DIMS):
    """Shard rows [rank*b/N, (rank+1)*b/N) of batch i = Rng(1+i) normal/integers."""
    from paper_2603_25976_b200.numeric import Rng

    bl = b_global // world
    out = []
    for i in range(n_batches):
        r = Rng(1 + i)
        X = r.normal(b_global * dims[0]).reshape(b_global, dims[0]).astype(np.float32)
        y = r.integers(b_global, dims[-1])
        out.append((X[rank * bl:(rank + 1) * bl], y[rank * bl:(rank + 1) * bl]))
    return out


def make_batches_fast(n_batches, b_global, rank, world, dims):
    """C5-sized batches (b x 3072 = 10^8 normals): numpy's PCG64 instead of the Python
    SplitMix64 stream, which would take minutes per batch; shard layout as make_batches."""
    bl = b_global // world
    out = []
    for i in range(n_batches):
        g = np.random.default_rng(1 + i)
        X = g.standard_normal((bl, dims[0]), dtype=np.float32) if world == 1 else \
            g.standard_normal((b_global, dims[0]), dtype=np.float32)[rank * bl:(rank + 1) * bl]
        y = g.integers(0, dims[-1], size=b_global)[rank * bl:(rank + 1) * bl] if world > 1 else \
            g.integers(0, dims[-1], size=bl)
        out.append((np.ascontiguousarray(X), y.astype(np.int64)))
    return out


def spec_c3():
    import paper_2603_25976_b200 as P

    return P.MethodSpec(curvature=P.CurvatureSpec("ggn_ce"),
                        solver=P.SolverSpec("cg", P.CgConfig(tol=1e-5, maxiter=10, stabilise_every=10,
                                                             warm_start=True)),
                        precond=P.PrecondSpec("diag_ema", 0.99), damping=P.DampingSpec("constant", 1.0),
                        estimator=P.EstimatorSpec("hutchinson", 1, every_k=10),
                        chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))


def spec_c4():
    import paper_2603_25976_b200 as P

    return P.MethodSpec(curvature=P.CurvatureSpec("ggn_ce"), solver=P.SolverSpec("row_cholesky"),
                        damping=P.DampingSpec("constant", 1.0),
                        chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))


def spec_c5():
    import paper_2603_25976_b200 as P

    return P.MethodSpec(curvature=P.CurvatureSpec("hessian"),
                        solver=P.SolverSpec("cg", P.CgConfig(tol=1e-5, maxiter=10, stabilise_every=10,
                                                             warm_start=True)),
                        damping=P.DampingSpec("constant", 1.0),
                        estimator=P.EstimatorSpec("hutchinson", 1, every_k=10),
                        telemetry=P.TelemetrySpec(trace_every_k=10, trace_probes=1),
                        chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))


SPECS = {"c3": spec_c3, "c4": spec_c4, "c5": spec_c5}

CADENCE_METRIC = ("newton_cg planned-step median ms, rho probes off (PAPER Table 3 workload: MLP 512-1024-1024-1, "
                  "b=256, HVP + CG maxiter 3, constant damping)")
CADENCE_KS = [-1, 10, 5, 2, 1]
CADENCE_DIMS = (512, 1024, 1024, 1)


def cadence_config(world):
    return {"workload": "cadence study (bench.py:135-207): newton_cg, synth_regression n=20000 d=512, "
                        "512-1024-1024-1 ReLU, b=256, constant lam=1, CG maxiter 3 warm start, "
                        "rho_every_k in {-1,10,5,2,1}, paired timing, window 50",
            "global_batch": 256, "dims": list(CADENCE_DIMS), "parallelism": f"replicas ({world})",
            "l2": "working set < L2 (latency-bound step; the paper's protocol, no flush)"}


def cpu_cadence_sample(steps, warmup, max_seconds=20.0):
    """The oracle's newton_cg step (rho off) on the cadence workload: median ms."""
    from oracle import curvopt_oracle as O

    (Xtr, ytr), _ = O.gen_regression(20000, 512, 0.1, 0)
    root = O.ORng(0)
    w = O.init_params(CADENCE_DIMS, "relu", root.split())
    bat = O.Batcher(Xtr, ytr, 256, root.split())
    spec = O.OSpec(curvature="hessian", maxiter=3, rho_every_k=-1)
    st = O.oracle_init(spec, w.size)
    times = []
    t_all = time.perf_counter()
    for i in range(steps + warmup):
        X, y = bat.next()
        t0 = time.perf_counter()
        w, st, _, _ = O.oracle_step(spec, CADENCE_DIMS, "relu", "mse", w, X, y, st)
        if i >= warmup:
            times.append((time.perf_counter() - t0) * 1e3)
        if time.perf_counter() - t_all > max_seconds and len(times) >= 3:
            break
    return float(np.median(times)), len(times)


def run_cadence(args, rank, world):
    """The cadence study on the device (replicas: rank 0 reports)."""
    import torch

    import paper_2603_25976_b200 as P
    from paper_2603_25976_b200 import harness as H
    from paper_2603_25976_b200.runtime import runtime

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    rt = runtime()
    window = min(50, args.steps)
    H.bench_cadence(CADENCE_KS, steps=4, window=4, warmup=2)  # allocator / plan warm-up
    from paper_2603_25976_b200.method import StepGraph

    launches0 = rt.launches() + StepGraph.replayed_kernels
    gc.collect()
    gc.disable()
    t_wall = time.perf_counter()
    with ClockSampler(dev.index) as clk:
        rows = H.bench_cadence(CADENCE_KS, steps=args.steps, window=window, warmup=args.warmup)
    wall = time.perf_counter() - t_wall
    launches = rt.launches() + StepGraph.replayed_kernels - launches0
    gc.enable()
    table = [{"rho_every_k": k, "median_ms": med, "p90_ms": p90, "overhead_pct": ov,
              "paper_median_ms": H.PAPER_TABLE3_MS[k][0], "paper_p90_ms": H.PAPER_TABLE3_MS[k][1]}
             for k, med, p90, ov in rows]
    med_off = rows[0][1]
    # e2e: the rho-off setting through the public API with host buffers (pinned batch in,
    # host parameters out every step), wall clock around the step as the protocol does
    train, _ = H.gen_regression(20000, 512, 0.1, 0)
    model = P.Model(512, (1024, 1024), 1, "relu")
    meth = H.cadence_methods([-1], model)[-1]
    root = P.Rng(0)
    w = P.init_params(model, root.split())
    w = P.ParamVector(torch.from_numpy(np.asarray(w.data, dtype=np.float32)).pin_memory(), w.layout)
    bat = H.EpochBatcher(train, 256, root.split())
    Xh = torch.from_numpy(np.ascontiguousarray(train.X, dtype=np.float32)).pin_memory()
    yh = torch.from_numpy(np.ascontiguousarray(train.y, dtype=np.float32)).pin_memory()
    st = meth.init(w, seed=0)
    et = []
    for t in range(args.steps + args.warmup):
        idx = torch.from_numpy(np.ascontiguousarray(bat.next_indices(), dtype=np.int64))
        b = P.Batch(Xh[idx].pin_memory(), yh[idx].pin_memory(), "mse")
        t0 = time.perf_counter()
        w, st, _ = meth.step(w, b, st)
        et.append((time.perf_counter() - t0) * 1e3)
    e2e_ms = H.timing_summary(et, args.warmup, window).median_ms
    # roofline of the dominant unit: one HVP at b=256 (the step's products), CUDA events
    wd = P.init_params(model, P.Rng(0)).to_device(dev)
    Xd = torch.from_numpy(np.ascontiguousarray(train.X[:256], dtype=np.float32)).to(dev)
    yd = torch.from_numpy(np.ascontiguousarray(train.y[:256], dtype=np.float32)).to(dev)
    snap = P.make_snapshot("hessian", model, wd, P.Batch(Xd, yd, "mse"))
    v = torch.randn(wd.dim, device=dev)
    out = torch.empty_like(v)
    for _ in range(5):
        snap.apply(1, v, out)
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for _ in range(50):
        snap.apply(1, v, out)
    g1.record(stream)
    torch.cuda.synchronize()
    hvp_ms = g0.elapsed_time(g1) / 50
    snap.close()
    flops = hvp_flops(CADENCE_DIMS, 256)
    try:
        peak = f16_peak_tflops() / 3.0
        peak_note = "measured cuBLAS fp16 / 3 (3xFP16 split passes)"
    except Exception:
        peak = measured_peaks().get("bf16_tflops", 1626.3) / 3
        peak_note = "MEASURED_PEAKS bf16 burst / 3"
    achieved = flops / (hvp_ms * 1e-3) / 1e12
    if rank != 0:
        return
    line = {"metric": CADENCE_METRIC, "value": med_off, "unit": "ms", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": med_off, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": med_off / H.PAPER_TABLE3_MS[-1][0],
            "vs_baseline_note": "value / 0.84 ms (PAPER Table 3, RTX A4000 JAX, rho off; BASELINE.md row 1)",
            "dtype": "f32 (scaled 3xFP16 tensor-core GEMMs, fp32 accumulate, fp64 reductions)",
            "data": "synthetic (reference gen_regression)", "config": cadence_config(world), "cadence": table,
            "wall_s_all_settings": wall,
            "e2e": {"value": e2e_ms, "unit": "ms", "h2d_bytes_per_step": 256 * 512 * 4 + 256 * 4 + wd.dim * 4,
                    "d2h_bytes_per_step": wd.dim * 4 + 24 * 8},
            "gpu_launches": launches, "clocks": clk.summary(),
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None, "traffic_source": None,
                         "unit_of_work": f"one HVP at b=256: {flops / 1e9:.2f} GFLOP useful, {hvp_ms * 1e3:.1f} us "
                                         f"avg over 50 (CUDA events); launch/latency-bound at this size",
                         "peak_source": peak_note}}
    if not args.no_cpu:
        med_cpu, n = cpu_cadence_sample(10, 2)
        line["cpu_baseline"] = {"value": med_cpu, "unit": "ms", "cores": host_cores(), "kind": "port",
                                "sample": f"{n} newton_cg steps (rho off) of the numpy/OpenBLAS f64 oracle, median",
                                "cpu_model": cpu_model()}
    print(json.dumps(line), flush=True)


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.first = threading.Event()
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi needs a moment to start: enter the timed region only once it samples
            self.first.wait(timeout=5.0)
        except Exception:
            self.proc = None
        self.start_idx = len(self.rows)
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)
                self.first.set()

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows[self.start_idx:] or self.rows[-1:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def product_traffic(key="c3"):
    """DRAM bytes of one product (C3 GGN / C5 HVP) from the committed ncu --set full
    capture, or None."""
    names = {"c3": ("r2_product_traffic.json", "r1d_product_traffic.json"), "c5": ("r2_c5_hvp_traffic.json",)}
    for name in names.get(key, ()):
        try:
            with open(os.path.join(ROOT, "profiles", name)) as f:
                return float(json.load(f)["dram_bytes_per_product"]), name
        except Exception:
            continue
    return None, None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def f16_peak_tflops():
    """Dense FP16 tensor-core peak on this box: cuBLAS fp16 8192^3 (fp32 accumulate), best of 5."""
    import torch

    a = torch.randn(8192, 8192, device="cuda", dtype=torch.float16)
    b = torch.randn(8192, 8192, device="cuda", dtype=torch.float16)
    for _ in range(2):
        a @ b
    best = 1e9
    for _ in range(5):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        a @ b
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return 2 * 8192**3 / (best * 1e-3) / 1e12


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ---------------------------------------------------------------------------
# CPU oracle (reference arm / cpu_baseline): the numpy restatement of the
# reference step, timed on the host cores (the reference itself is pure Python
# and does not travel to the GPU box).
# ---------------------------------------------------------------------------
def cpu_c3_steps(steps, warmup, max_seconds):
    from oracle import curvopt_oracle as O

    spec = O.OSpec(precond="diag_ema", estimator_every_k=10)
    w = O.init_params(DIMS, "relu", O.ORng(0))
    batches = [(X.astype(np.float64), y) for X, y in make_batches(2, GLOBAL_B, 0, 1)]
    st = O.oracle_init(spec, w.size)
    for i in range(warmup):
        w, st, _, _ = O.oracle_step(spec, DIMS, "relu", "ce", w, *batches[i % 2], st)
    times, gv_log = [], []
    t_all = time.perf_counter()
    for i in range(steps):
        t0 = time.perf_counter()
        w, st, _, _ = O.oracle_step(spec, DIMS, "relu", "ce", w, *batches[(warmup + i) % 2], st, gv_log=gv_log)
        times.append(time.perf_counter() - t0)
        if time.perf_counter() - t_all > max_seconds:
            break
    return len(times) / sum(times), times, gv_log


def cpu_gv_rate(threads, b=GLOBAL_B, n=2):
    """GGN products/s of the oracle at b rows with `threads` BLAS threads."""
    from threadpoolctl import threadpool_limits

    from oracle import curvopt_oracle as O

    w = O.init_params(DIMS, "relu", O.ORng(0))
    X, y = O.synthetic_batch(b, DIMS[0], DIMS[-1])
    with threadpool_limits(limits=threads):
        lin = O.linearize(DIMS, "relu", "ce", w, X, y)
        v = O.ORng(2).normal(w.size)
        O.ggn_matvec(lin, v)
        t0 = time.perf_counter()
        for _ in range(n):
            O.ggn_matvec(lin, v)
        return n / (time.perf_counter() - t0)


def cpu_row_sample(wl, threads):
    """Bounded sample of the C4 row lane on the oracle: Gram + Cholesky + backprojection at
    b=1024 (m=10240), extrapolated to b=4096 by the flop model (Gram ~ m^2, potrf ~ m^3)."""
    from threadpoolctl import threadpool_limits

    from oracle import curvopt_oracle as O

    bs = 1024
    dims = wl.dims
    w = O.init_params(dims, "relu", O.ORng(0))
    X, y = O.synthetic_batch(bs, dims[0], dims[-1])
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        lin = O.linearize(dims, "relu", "ce", w, X, y)
        seeds, rhs = O.row_seeds_rhs(lin)
        t1 = time.perf_counter()
        gram = O.output_gram(lin, seeds)
        t2 = time.perf_counter()
        v = O.row_cholesky(gram, rhs, float(bs))
        t3 = time.perf_counter()
        O.row_transpose(lin, seeds, v)
        t4 = time.perf_counter()
    k = wl.b / bs
    est = (t1 - t0 + t4 - t3) * k + (t2 - t1) * k * k + (t3 - t2) * k ** 3
    return 1.0 / est, f"b={bs} (m={bs * dims[-1]}) oracle row step {t4 - t0:.2f} s, extrapolated to b={wl.b} " \
                      f"by the flop model (linearize/backprojection x{k:.0f}, Gram x{k * k:.0f}, potrf x{k ** 3:.0f})"


def cpu_hvp_sample(wl, threads):
    """Bounded sample of the C5 step: one oracle HVP at b=512 rows, extrapolated linearly to
    b=32768 and to the products of a planned step (CG 10 + warm start + probes)."""
    from threadpoolctl import threadpool_limits

    from oracle import curvopt_oracle as O

    bs = 512
    dims = wl.dims
    w = O.init_params(dims, "relu", O.ORng(0))
    X, y = O.synthetic_batch(bs, dims[0], dims[-1])
    with threadpool_limits(limits=threads):
        t0 = time.perf_counter()
        lin = O.linearize(dims, "relu", "ce", w, X, y)
        t1 = time.perf_counter()
        O.hvp(lin, O.ORng(2).normal(w.size))
        t2 = time.perf_counter()
    k = wl.b / bs
    products = 11.1  # measured products per planned C5 step on the device run (CG 10 + warm start + probes / 10)
    est = k * ((t1 - t0) + products * (t2 - t1))
    return 1.0 / est, f"b={bs} oracle linearize {t1 - t0:.2f} s + one HVP {t2 - t1:.2f} s, extrapolated x{k:.0f} " \
                      f"rows and x{products} products per step"


def run_reference(args, rank, world):
    """The reference arm: the CPU restatement of curvopt's step on the host cores."""
    if rank != 0:
        return
    if args.config == "cadence":
        med, n = cpu_cadence_sample(args.steps, args.warmup, max_seconds=120.0)
        cores = host_cores()
        print(json.dumps({"impl": "reference", "metric": CADENCE_METRIC, "value": med, "unit": "ms",
                          "n_gpus": world, "steps": n, "warmup": args.warmup, "ms_per_step": med,
                          "higher_is_better": False, "scaling": "weak", "vs_baseline": med / 0.84,
                          "dtype": "f64", "data": "synthetic (reference gen_regression)",
                          "config": cadence_config(world),
                          "cpu_baseline": {"value": med, "unit": "ms", "cores": cores, "kind": "port",
                                           "sample": f"{n} newton_cg steps (rho off), oracle port, median",
                                           "cpu_model": cpu_model()},
                          "e2e": {"value": med, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}),
              flush=True)
        return
    wl = WORKLOADS[args.config]
    cores = host_cores()
    if wl.key == "c3":
        sps, times, gv = cpu_c3_steps(args.steps, args.warmup, max_seconds=240.0)
        sample = (f"{len(times)} full C3 planned steps (after {args.warmup} warm-up) of the numpy/OpenBLAS f64 "
                  f"oracle restating curvopt Method.step; {cores} BLAS threads. The reference's own ggn_ce "
                  f"snapshot also runs a per-example eigh (curvature.py:118-119) the port skips, so the port is "
                  f"the faster of the two")
        gvps = sum(gv) / sum(times) if gv else None
        steps = len(times)
    elif wl.key == "c4":
        sps, sample = cpu_row_sample(wl, cores)
        gvps, steps = None, args.steps
    else:
        sps, sample = cpu_hvp_sample(wl, cores)
        gvps, steps = None, args.steps
    line = {"impl": "reference", "metric": wl.metric, "value": sps, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": args.warmup, "ms_per_step": 1e3 / sps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": wl.config(world), "gv_per_s": gvps,
            "cpu_baseline": {"value": sps, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                             "cpu_model": cpu_model()},
            "e2e": {"value": sps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# The GPU arm
# ---------------------------------------------------------------------------
def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2603_25976_b200 as P
    from paper_2603_25976_b200.runtime import runtime

    wl = WORKLOADS[args.config]
    dims = wl.dims
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    rt = runtime()
    model = P.Model(dims[0], dims[1:-1], dims[-1], "relu")
    meth = P.assemble(SPECS[wl.key](), model)
    w0 = P.init_params(model, P.Rng(0))
    # batch-sharded on every lane; the row lane's solve is the distributed block-cyclic
    # Cholesky (RowOps gathers the batch for the whole-batch D chain and back-projection)
    shard_world, shard_rank = world, rank
    row = wl.lane == "row"
    bl = wl.b // shard_world
    nb = 4 if wl.key == "c3" else 2
    if wl.key == "c3":
        host_batches = make_batches(nb, wl.b, shard_rank, shard_world, dims)
    else:
        host_batches = make_batches_fast(nb, wl.b, shard_rank, shard_world, dims)

    def mk_batch(X, y):
        return P.Batch(X, y, "ce", global_size=wl.b, row_offset=shard_rank * bl)

    dev_batches = [mk_batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev)) for X, y in host_batches]
    w = w0.to_device(dev)
    st = meth.init(w, 0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        w, st, info = meth.step(w, dev_batches[i % nb], st)
    stream = torch.cuda.current_stream()
    gv_total = 0
    from paper_2603_25976_b200.method import StepGraph

    launches0 = rt.launches() + StepGraph.replayed_kernels
    # no cyclic-GC pause inside the timed regions (a full collection is tens of ms, which
    # the step's single host sync would expose as GPU idle)
    gc.collect()
    gc.freeze()
    gc.disable()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            w, st, info = meth.step(w, dev_batches[(args.warmup + i) % nb], st)
            gv_total += getattr(meth, "last_products", 0)
        ev1.record(stream)
        barrier()
    launches = rt.launches() + StepGraph.replayed_kernels - launches0  # eager launches + replayed graph kernels
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    sps = args.steps / (ms * 1e-3)
    gv_per_s = gv_total / (ms * 1e-3)

    # ---- e2e: the same steps through the public API, inputs from pinned host memory ----
    # (a) training-loop form: parameters stay device-resident across steps (as in any GPU
    #     training loop); every step's batch comes from pinned host memory through the
    #     public BatchPrefetcher (H2D on a copy stream, overlapping the previous step) and
    #     the step's result (the StepInfo scalar block) is read back to the host.
    from paper_2603_25976_b200.pipeline import BatchPrefetcher

    pinned = [(torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory()) for X, y in host_batches]
    counter = [0]

    def source():
        b = pinned[counter[0] % nb]
        counter[0] += 1
        return b

    pf = BatchPrefetcher(source, "ce", global_size=wl.b, row_offset=shard_rank * bl, device=dev)
    we = w0.to_device(dev)
    st_e = meth.init(we, 0)
    for i in range(min(3, args.warmup)):
        we, st_e, _ = meth.step(we, pf.next(), st_e)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        we, st_e, info_e = meth.step(we, pf.next(), st_e)
    e1.record(stream)
    barrier()
    ems = e0.elapsed_time(e1)
    te = torch.tensor([ems], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    ems = float(te.item())
    h2d = pf.h2d_bytes
    d2h = 24 * 8  # the step's scalar block (StepInfo)
    e2e = {"value": args.steps / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "form": "device-resident parameters; batch H2D from pinned host memory via BatchPrefetcher "
                   "(overlapped with the previous step); StepInfo D2H"}
    # (b) host-parameter form: w from and w' back to pinned host memory every step as well
    wh = P.ParamVector(torch.from_numpy(np.asarray(w.data.cpu().numpy())).pin_memory(), w.layout)
    st_h = meth.init(w, 0)
    for i in range(min(2, args.warmup)):
        wh, st_h, _ = meth.step(wh, mk_batch(*pinned[i % nb]), st_h)
    barrier()
    h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0.record(stream)
    for i in range(args.steps):
        wh, st_h, _ = meth.step(wh, mk_batch(*pinned[i % nb]), st_h)
    h1.record(stream)
    barrier()
    hms = h0.elapsed_time(h1)
    th = torch.tensor([hms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(th, op=dist.ReduceOp.MAX)
    hms = float(th.item())
    e2e_host = {"value": args.steps / (hms * 1e-3), "unit": UNIT,
                "h2d_bytes_per_step": bl * dims[0] * 4 + bl * 8 + w.dim * 4, "d2h_bytes_per_step": w.dim * 4 + 24 * 8}
    gc.enable()

    # ---- roofline of the dominant unit, timed live with CUDA events on the launch stream ----
    try:
        f16 = f16_peak_tflops() if rank == 0 else None
        peak = f16 / 3.0 if f16 else None
        peak_note = f"measured cuBLAS fp16 {f16:.0f} TF/s / 3 (3xFP16 split passes)" if f16 else None
    except Exception:
        peak = measured_peaks().get("bf16_tflops", 1626.3) / 3
        peak_note = "MEASURED_PEAKS bf16 burst / 3 (3xFP16 split passes)"
    if row:
        flops = row_flops(dims, wl.b)
        achieved = flops / (ms / args.steps * 1e-3) / 1e12 / world
        unit_note = (f"one row-lane planned step at b={wl.b} (m={wl.b * dims[-1]}): Gram as SYRK + potrf = "
                     f"{flops / 1e12:.2f} TFLOP useful, {ms / args.steps:.1f} ms/step (CUDA events)"
                     + (f", per GPU of {world}" if world > 1 else ""))
        traffic, tsrc = None, None
    else:
        kind = 1 if wl.kind == "hessian" else 0
        snap = P.make_snapshot("hessian" if kind else "ggn_ce", model, w, dev_batches[0])
        v = torch.randn(w.dim, device=dev)
        out = torch.empty_like(v)
        for _ in range(3):
            snap.apply(kind, v, out)
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n_gv = 20 if wl.key == "c3" else 5
        g0.record(stream)
        for _ in range(n_gv):
            snap.apply(kind, v, out)
        g1.record(stream)
        torch.cuda.synchronize()
        gv_ms = g0.elapsed_time(g1) / n_gv
        snap.close()
        flops = hvp_flops(dims, bl) if kind else gv_flops(dims, bl)
        achieved = flops / (gv_ms * 1e-3) / 1e12
        unit_note = (f"one {'HVP' if kind else 'GGN'} product at b={bl}: {flops / 1e9:.1f} GFLOP useful, "
                     f"{gv_ms:.3f} ms avg over {n_gv} (CUDA events)")
        traffic, tsrc = product_traffic(wl.key)

    if rank != 0:
        return
    clocks = clk.summary()
    line = {"metric": wl.metric, "value": sps, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32 (scaled 3xFP16 tensor-core GEMMs, fp32 accumulate, fp64 reductions)",
            "data": "synthetic", "config": wl.config(world),
            "gv_per_s": gv_per_s if not row else None, "gv_per_step": gv_total / args.steps if not row else None,
            "e2e": e2e, "e2e_host_params": e2e_host, "gpu_launches": launches, "clocks": clocks,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": traffic,
                         "traffic_source": f"profiles/{tsrc} (ncu --set full, DRAM read+write bytes summed over "
                                           f"the product's kernels)" if tsrc else None,
                         "unit_of_work": unit_note, "peak_source": peak_note}}
    if world == 1 and not args.no_cpu:
        cores = host_cores()
        if wl.key == "c3":
            sps_cpu, times, _ = cpu_c3_steps(3, 0, max_seconds=15.0)
            sample = f"{len(times)} full C3 planned steps of the numpy/OpenBLAS f64 oracle, {cores} BLAS threads"
            extra = {"gv_per_s_1thread": cpu_gv_rate(1), "gv_per_s_all_threads": cpu_gv_rate(cores),
                     "gv_sample": f"2 oracle GGN products at b={wl.b} with OPENBLAS threads = 1 and = {cores}"}
        elif wl.key == "c4":
            sps_cpu, sample = cpu_row_sample(wl, cores)
            extra = {}
        else:
            sps_cpu, sample = cpu_hvp_sample(wl, cores)
            extra = {}
        line["cpu_baseline"] = {"value": sps_cpu, "unit": UNIT, "cores": cores, "kind": "port", "sample": sample,
                                "cpu_model": cpu_model(), **extra}
    print(json.dumps(line), flush=True)


def _rank_main(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if world > 1:
        import torch
        import torch.distributed as dist

        if os.environ.get("CURVOPT_BENCH_SHARED_GPU") == "1":
            # test hook: every rank on cuda:0 over gloo (the library's host communicator) --
            # the multi-rank bench flow on a one-GPU box; numbers from it are not bench values
            os.environ["LOCAL_RANK"] = "0"
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
            dist.init_process_group("nccl")
    try:
        if args.config == "cadence":
            run_cadence(args, rank, world)
        else:
            run_ours(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()


def _spawn_entry(local_rank, args, world, port):
    os.environ.update(RANK=str(local_rank), LOCAL_RANK=str(local_rank), WORLD_SIZE=str(world),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    _rank_main(args)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(WORKLOADS) + ["cadence"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        raise SystemExit("bench.py: --warmup must be >= 3")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # launch the N ranks ourselves (one process per GPU), as torchrun would
        import torch
        import torch.multiprocessing as mp

        if torch.cuda.device_count() < args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but only {torch.cuda.device_count()} visible")
        port = 29000 + os.getpid() % 2000
        mp.spawn(_spawn_entry, args=(args, args.gpus, port), nprocs=args.gpus, join=True)
        return
    _rank_main(args)


if __name__ == "__main__":
    main()
