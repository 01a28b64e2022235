"""Benchmark: GGN + PCG planned steps/sec (and Gv products/sec) on B200.

Workload (BASELINE.json configs[2], "C3"): MLP 784-1024-1024-10 softmax-CE, global
batch 8192, GGN curvature, PCG (tol 1e-5, maxiter 10, stabilise 10, warm start)
with the diag-EMA(0.99) preconditioner fed by a Hutchinson probe every 10 steps,
constant damping lam = 1, chain (scale 1e-3, scale -1).  Synthetic data from the
reference's SplitMix64 stream (MNIST-shaped), random-init weights (init_params).
With N GPUs the global batch is sharded b/N per rank (strong scaling); every Gv
and gradient is NCCL all-reduced inside the native library.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).
"""

from __future__ import annotations

import argparse
import gc
import json
import math
import os
import subprocess
import sys
import threading
import time

if "OPENBLAS_NUM_THREADS" not in os.environ:
    try:
        os.environ["OPENBLAS_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    except Exception:
        pass

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DIMS = (784, 1024, 1024, 10)
GLOBAL_B = 8192
METRIC = "GGN-CG planned steps/sec (C3: 784-1024-1024-10, b=8192, PCG + diag-EMA)"
UNIT = "steps/s"


def P_w(dims):
    return sum(dims[i] * dims[i + 1] for i in range(len(dims) - 1))


def gv_flops(dims, b):
    """Useful fp32-equivalent flops of one GGN product: 8 b P_w - 4 b n0 n1."""
    return 8 * b * P_w(dims) - 4 * b * dims[0] * dims[1]


def make_batches(n_batches, b_global, rank, world):
    """Shard rows [rank*b/N, (rank+1)*b/N) of batch i = Rng(1+i) normal/integers."""
    from paper_2603_25976_b200.numeric import Rng

    bl = b_global // world
    out = []
    for i in range(n_batches):
        r = Rng(1 + i)
        X = r.normal(b_global * DIMS[0]).reshape(b_global, DIMS[0]).astype(np.float32)
        y = r.integers(b_global, DIMS[-1])
        out.append((X[rank * bl:(rank + 1) * bl], y[rank * bl:(rank + 1) * bl]))
    return out


def spec_c3():
    import paper_2603_25976_b200 as P

    return P.MethodSpec(curvature=P.CurvatureSpec("ggn_ce"),
                        solver=P.SolverSpec("cg", P.CgConfig(tol=1e-5, maxiter=10, stabilise_every=10,
                                                             warm_start=True)),
                        precond=P.PrecondSpec("diag_ema", 0.99), damping=P.DampingSpec("constant", 1.0),
                        estimator=P.EstimatorSpec("hutchinson", 1, every_k=10),
                        chain=(P.transforms.scale(1e-3), P.transforms.scale(-1.0)))


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
            # (a short timed region could otherwise see no sample at all)
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
        # samples taken inside the timed region (else the one just before it)
        rows = self.rows[self.start_idx:] or self.rows[-1:]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        self.rows = rows
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def product_traffic():
    """DRAM bytes of one GGN product from the committed ncu --set full capture
    (scratch/product_traffic.py -> profiles/r1d_product_traffic.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1d_product_traffic.json")) as f:
            return float(json.load(f)["dram_bytes_per_product"])
    except Exception:
        return None


# the tensor-core launches of one C3 product in the committed capture's order
_GEMM_ROLES = [("JVP0 X V0, mask bits", 8192, 1024, 785), ("JVP1 [A1|da0][V1;W1] + fused output JVP", 8192, 1024, 2049),
               ("dW1 weight gradient, split-K, side stream (SM share)", 1025, 1024, 8192),
               ("dX1 backward, mask bits (SM share)", 8192, 1024, 1024), ("dW0 weight gradient, split-K", 785, 1024, 8192)]


def gemm_launch_rooflines(peak):
    """Per-launch tensor roofline of the product's GEMMs from the committed ncu --set full
    capture (cold-cache serialised replay: co-scheduled launches replay on their SM share)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r1d_product_traffic.json")) as f:
            kern = json.load(f)["kernels"]
    except Exception:
        return None
    tc2 = [k for k in kern if "k_gemm_tc2" in k["kernel"]]
    if len(tc2) != len(_GEMM_ROLES):
        return None
    out = []
    for k, (role, m, n, kk) in zip(tc2, _GEMM_ROLES):
        tf = 2.0 * m * n * kk / (k["us"] * 1e-6) / 1e12
        out.append({"launch": role, "useful_gflop": round(2.0 * m * n * kk / 1e9, 2), "us": k["us"],
                    "tflops": round(tf, 1), "frac": round(tf / peak, 3) if peak else None,
                    "tensor_pipe_pct": k.get("tensor_pipe_pct"),
                    "dram_bytes": k["dram_read_B"] + k["dram_write_B"]})
    return out


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


# ---------------------------------------------------------------------------
# CPU oracle (reference arm / cpu_baseline): the numpy restatement of the
# reference step, timed on the host cores.
# ---------------------------------------------------------------------------
def cpu_oracle_run(max_seconds=20.0, max_steps=None, warmup=1):
    from oracle import curvopt_oracle as O

    spec = O.OSpec(precond="diag_ema", estimator_every_k=10)
    w = O.init_params(DIMS, "relu", O.ORng(0))
    batches = []
    for i in range(2):
        r = O.ORng(1 + i)
        X = r.normal(GLOBAL_B * DIMS[0]).reshape(GLOBAL_B, DIMS[0])
        batches.append((X, r.integers(GLOBAL_B, DIMS[-1])))
    st = O.oracle_init(spec, w.size)
    gv_log = []
    for i in range(warmup):
        w, st, _, _ = O.oracle_step(spec, DIMS, "relu", "ce", w, *batches[i % 2], st)
    times = []
    gv_log = []
    t_all = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        w, st, info, _ = O.oracle_step(spec, DIMS, "relu", "ce", w, *batches[len(times) % 2], st, gv_log=gv_log)
        times.append(time.perf_counter() - t0)
        if max_steps is not None and len(times) >= max_steps:
            break
        if time.perf_counter() - t_all > max_seconds:
            break
    sps = len(times) / sum(times)
    return sps, times, gv_log


def cores_used():
    try:
        return int(os.environ.get("OPENBLAS_NUM_THREADS") or len(os.sched_getaffinity(0)))
    except Exception:
        return os.cpu_count()


def run_reference(args, rank, world):
    if rank != 0:
        return
    W = min(args.warmup, 1)
    sps, times, gv = cpu_oracle_run(max_seconds=min(90.0, 20.0 * max(args.steps, 1)), max_steps=args.steps,
                                    warmup=W)
    sample = (f"{len(times)} full C3 planned steps (after {W} warm-up) of the numpy/OpenBLAS f64 oracle restating "
              f"curvopt Method.step; {cores_used()} BLAS threads")
    line = {"impl": "reference", "metric": METRIC, "value": sps, "unit": UNIT, "n_gpus": world,
            "steps": len(times), "warmup": W, "ms_per_step": 1e3 / sps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "C3 784-1024-1024-10 softmax-CE, GGN + PCG(diag-EMA 0.99, Hutchinson@10)",
                       "global_batch": GLOBAL_B, "parallelism": "host cores"},
            "gv_per_s": sum(gv) / sum(times) if gv else None,
            "cpu_baseline": {"value": sps, "unit": UNIT, "cores": cores_used(), "kind": "port", "sample": sample},
            "e2e": {"value": sps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world):
    import torch
    import torch.distributed as dist

    import paper_2603_25976_b200 as P
    from paper_2603_25976_b200.runtime import runtime

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    rt = runtime()
    model = P.Model(DIMS[0], DIMS[1:-1], DIMS[-1], "relu")
    meth = P.assemble(spec_c3(), model)
    w0 = P.init_params(model, P.Rng(0))
    bl = GLOBAL_B // world
    host_batches = make_batches(4, GLOBAL_B, rank, world)
    dev_batches = [P.Batch(torch.from_numpy(X).to(dev), torch.from_numpy(y).to(dev), "ce", global_size=GLOBAL_B)
                   for X, y in host_batches]
    w = w0.to_device(dev)
    st = meth.init(w, 0)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up (also triggers every lazy allocation)
    for i in range(args.warmup):
        w, st, info = meth.step(w, dev_batches[i % len(dev_batches)], st)
    # Gv counter: CG products + Hutchinson probes are read from the step records
    stream = torch.cuda.current_stream()
    gv_total = 0
    launches0 = rt.launches()
    # no cyclic-GC pause inside the timed regions (a full collection of the interpreter's
    # heap is tens of ms, which the step's single host sync would expose as GPU idle)
    gc.collect()
    gc.freeze()
    gc.disable()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    infos = []
    with ClockSampler(dev.index) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            w, st, info = meth.step(w, dev_batches[(args.warmup + i) % len(dev_batches)], st)
            infos.append(info)
            gv_total += meth.last_products
        ev1.record(stream)
        barrier()
    launches = rt.launches() - launches0
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    sps = args.steps / (ms * 1e-3)
    gv_per_s = gv_total / (ms * 1e-3)

    # ---- e2e: same steps through the public API with host (pinned) buffers ----
    e2e = None
    wh = P.ParamVector(torch.from_numpy(np.asarray(w.data.cpu().numpy())).pin_memory(), w.layout)
    pinned = [(torch.from_numpy(X).pin_memory(), torch.from_numpy(y).pin_memory()) for X, y in host_batches]
    st_e = meth.init(w, 0)
    for i in range(2):
        wh, st_e, _ = meth.step(wh, P.Batch(*pinned[i % 4], "ce", global_size=GLOBAL_B), st_e)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(args.steps):
        wh, st_e, _ = meth.step(wh, P.Batch(*pinned[i % 4], "ce", global_size=GLOBAL_B), st_e)
    e1.record(stream)
    barrier()
    ems = e0.elapsed_time(e1)
    te = torch.tensor([ems], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    ems = float(te.item())
    h2d = bl * DIMS[0] * 4 + bl * 8 + w.dim * 4
    d2h = w.dim * 4 + 16 * 8 + 48
    e2e = {"value": args.steps / (ems * 1e-3), "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h}

    gc.enable()
    # ---- roofline of the dominant unit: the GGN product (its GEMMs), timed live ----
    snap = P.make_snapshot("ggn_ce", model, w, dev_batches[0])
    v = torch.randn(w.dim, device=dev)
    out = torch.empty_like(v)
    for _ in range(3):
        snap.apply(0, v, out)
    barrier()
    g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n_gv = 20
    g0.record(stream)
    for _ in range(n_gv):
        snap.apply(0, v, out)
    g1.record(stream)
    torch.cuda.synchronize()
    gv_ms = g0.elapsed_time(g1) / n_gv
    snap.close()
    flops = gv_flops(DIMS, bl)
    achieved = flops / (gv_ms * 1e-3) / 1e12
    peaks = measured_peaks()
    # every useful flop of the product costs 3 fp16 tensor-core flops (hi.hi + hi.lo + lo.hi)
    try:
        f16 = f16_peak_tflops() if rank == 0 else None
        peak = f16 / 3.0 if f16 else None
        peak_note = f"measured cuBLAS fp16 {f16:.0f} TF/s / 3 (3xFP16 split passes)"
    except Exception:
        peak = peaks.get("bf16_tflops", 1626.3) / 3
        peak_note = "MEASURED_PEAKS bf16 burst / 3 (3xFP16 split passes)"

    if rank != 0:
        return
    clocks = clk.summary()
    line = {"metric": METRIC, "value": sps, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32 (scaled 3xFP16 tensor-core GEMMs, fp32 accumulate, fp64 reductions)", "data": "synthetic",
            "config": {"workload": "C3 784-1024-1024-10 softmax-CE, GGN + PCG(diag-EMA 0.99, Hutchinson@10), "
                                   "lam=1, CG tol 1e-5 maxiter 10", "global_batch": GLOBAL_B,
                       "parallelism": f"dp{world}", "l2": "per-step working set ~0.6 GB > 126 MB L2 (no flush)"},
            "gv_per_s": gv_per_s, "gv_per_step": gv_total / args.steps,
            "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak if peak else None, "traffic": product_traffic(),
                         "traffic_source": "profiles/r1d_product_traffic.json (ncu --set full, DRAM read+write "
                                           "bytes summed over the product's kernels, cold-cache replay)",
                         "unit_of_work": f"one GGN product at b={bl}: {flops / 1e9:.1f} GFLOP useful, "
                                         f"{gv_ms:.3f} ms avg over {n_gv} (CUDA events)",
                         "peak_source": peak_note,
                         "per_launch_ncu": gemm_launch_rooflines(peak) if bl == 8192 else None},
            "engine": os.environ.get("CURVOPT_ENGINE", "auto")}
    if world == 1 and not args.no_cpu:
        sps_cpu, times, gv = cpu_oracle_run(max_seconds=15.0, max_steps=3, warmup=0)
        line["cpu_baseline"] = {"value": sps_cpu, "unit": UNIT, "cores": cores_used(), "kind": "port",
                                "sample": f"{len(times)} full C3 planned steps of the numpy/OpenBLAS f64 oracle, "
                                          f"{cores_used()} BLAS threads"}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        dist.init_process_group("nccl")
    run_ours(args, rank, world)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
