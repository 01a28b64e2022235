"""Training / timing harness on the GPU (curvopt/harness: data.py:28-90, run.py:31-294,
bench.py:135-207 of the reference), for the planned step this package accelerates.

* Synthetic datasets restated from the reference generators (same `Rng` streams, so the
  same samples): `gen_regression`, `gen_classification`.  The dataset is copied to the
  device once; `EpochBatcher` draws the reference's epoch permutations on the host and
  gathers each batch on the device.
* `run_training` times `Method.step` with a monotonic clock around the step only
  (batching excluded), window means after warm-up (`timing_summary`), as the reference.
  `Method.step` ends in one device->host read of the step's scalars, so the wall clock
  around it covers the device work.
* `bench_cadence` is the paper's only published measurement of this path (Table 3,
  PAPER.md:839-880): newton_cg on MLP 512-1024-1024-1 at b = 256 with constant damping
  and a fixed CG budget, sweeping `rho_every_k` over {-1, 10, 5, 2, 1}, paired timing
  (every step runs once per setting from the same buffers, in rotating order).

The data-file reader (IDX), CSV/meta output beyond the cadence table and the other
studies are outside the accelerated path (SURVEY §2 out of scope).
"""

from __future__ import annotations

import json
import time
from dataclasses import asdict, dataclass
from pathlib import Path

import numpy as np
import torch

from .errors import ContractError
from .method import Method, make
from .models import Batch, Model, init_params
from .numeric import Rng
from .runtime import runtime
from .telemetry import STEP_INFO_FIELDS


# -- datasets (data.py:28-90) ---------------------------------------------------------
@dataclass(frozen=True)
class Dataset:
    X: np.ndarray
    y: np.ndarray
    loss_kind: str  # "mse" | "ce"
    n_classes: int | None = None

    @property
    def n(self) -> int:
        return self.X.shape[0]

    @property
    def input_dim(self) -> int:
        return self.X.shape[1]


def _split(X, y, loss_kind, n_classes, train_frac):
    n_train = int(X.shape[0] * train_frac)
    return (Dataset(X[:n_train], y[:n_train], loss_kind, n_classes),
            Dataset(X[n_train:], y[n_train:], loss_kind, n_classes))


def gen_regression(n: int, d: int, noise_std: float, seed: int, train_frac: float = 0.9):
    """Linear teacher y = X beta + noise on an iid gaussian design (data.py:51-60)."""
    rng = Rng(seed)
    X = rng.normal(n * d).reshape(n, d)
    beta = rng.normal(d)
    noise = rng.normal(n) * noise_std
    return _split(X, (X @ beta + noise)[:, None], "mse", None, train_frac)


def gen_classification(n: int, d: int, classes: int, separation: float, seed: int, train_frac: float = 0.9):
    """Balanced gaussian blobs, class means on the signed axes (data.py:63-90)."""
    if classes < 2:
        raise ValueError("gen_classification requires classes >= 2")
    rng = Rng(seed)
    means = np.zeros((classes, d))
    for k in range(classes):
        if k < 2 * d:
            means[k, k // 2] = (separation / 2.0) * (1.0 if k % 2 == 0 else -1.0)
        else:
            u = rng.normal(d)
            means[k] = (separation / 2.0) * u / np.linalg.norm(u)
    labels = (np.arange(n) % classes)[rng.permutation(n)]
    X = means[labels] + rng.normal(n * d).reshape(n, d)
    return _split(X, labels.astype(np.int64), "ce", classes, train_frac)


class DeviceDataset:
    """A dataset resident in device memory (inputs fp32, targets fp32 / int64)."""

    def __init__(self, ds: Dataset, device=None):
        dev = device if device is not None else runtime().device
        self.ds = ds
        self.X = torch.from_numpy(np.ascontiguousarray(ds.X, dtype=np.float32)).to(dev)
        if ds.loss_kind == "ce":
            self.y = torch.from_numpy(np.ascontiguousarray(ds.y, dtype=np.int64)).to(dev)
        else:
            self.y = torch.from_numpy(np.ascontiguousarray(ds.y, dtype=np.float32)).to(dev)
        self.loss_kind = ds.loss_kind

    @property
    def n(self) -> int:
        return self.ds.n


class EpochBatcher:
    """Fixed-size batches from precomputed epoch permutations (run.py:174-192).

    The permutations are the reference's (host `Rng`); the rows are gathered on the
    device, so a batch never crosses PCIe."""

    def __init__(self, ds, batch_size: int, rng: Rng):
        self.dd = ds if isinstance(ds, DeviceDataset) else DeviceDataset(ds)
        if batch_size > self.dd.n:
            raise ContractError("batch_size exceeds dataset size")
        self.batch_size = batch_size
        self.rng = rng
        self._perm = rng.permutation(self.dd.n)
        self._pos = 0

    def next_indices(self) -> np.ndarray:
        if self._pos + self.batch_size > self.dd.n:
            self._perm = self.rng.permutation(self.dd.n)
            self._pos = 0
        idx = self._perm[self._pos:self._pos + self.batch_size]
        self._pos += self.batch_size
        return idx

    def next(self) -> Batch:
        hidx = np.ascontiguousarray(self.next_indices(), dtype=np.int64)
        idx = torch.from_numpy(hidx).to(self.dd.X.device)
        hint = {}
        if self.dd.loss_kind == "ce":  # label-range contract from the host labels: no device read
            yh = self.dd.ds.y[hidx]
            hint = {"_ymin": int(yh.min()), "_ymax": int(yh.max())}
        return Batch(self.dd.X.index_select(0, idx), self.dd.y.index_select(0, idx), self.dd.loss_kind, _dev=hint)


# -- run configuration and timing (run.py:31-110) -------------------------------------
@dataclass(frozen=True)
class TimingConfig:
    warmup_steps: int = 2
    window: int = 100

    def __post_init__(self):
        if self.warmup_steps < 1 or self.window < 1:
            raise ContractError("warmup_steps and window must be >= 1")


@dataclass(frozen=True)
class RunConfig:
    dataset: dict
    model: dict
    method: dict
    steps: int
    batch_size: int
    seed: int = 0
    timing: TimingConfig = TimingConfig()

    def to_dict(self) -> dict:
        return asdict(self)


@dataclass(frozen=True)
class TimingSummary:
    window_means_ms: tuple[float, ...]
    median_ms: float
    mean_ms: float
    std_ms: float
    p90_ms: float


@dataclass
class RunResult:
    step_rows: list[list]
    timing: TimingSummary
    final_w: object = None


def timing_summary(step_times_ms, warmup_steps: int, window: int) -> TimingSummary:
    """Window means over post-warmup steps; run stats over the window means (run.py:95-110)."""
    timed = np.asarray(step_times_ms[warmup_steps:], dtype=np.float64)
    if timed.size == 0:
        return TimingSummary((), float("nan"), float("nan"), float("nan"), float("nan"))
    means = [float(timed[lo:lo + window].mean()) for lo in range(0, timed.size, window)]
    return TimingSummary(tuple(means), float(np.median(means)), float(np.mean(means)), float(np.std(means)),
                         float(np.percentile(means, 90)))


def build_dataset(cfg: dict):
    kind = cfg["kind"]
    p = dict(cfg.get("params", {}))
    if kind == "synth_regression":
        return gen_regression(int(p.get("n", 20000)), int(p.get("d", 128)), float(p.get("noise_std", 0.1)),
                              int(p.get("seed", 0)))
    if kind == "synth_classification":
        return gen_classification(int(p.get("n", 20000)), int(p.get("d", 32)), int(p.get("classes", 10)),
                                  float(p.get("separation", 10.0)), int(p.get("seed", 0)))
    raise ContractError(f"unknown dataset kind {kind!r}")


def build_model(cfg: dict) -> Model:
    return Model(int(cfg["input_dim"]), tuple(int(h) for h in cfg["hidden"]), int(cfg["output_dim"]),
                 cfg.get("activation", "relu"))


def build_method(cfg: dict, model: Model) -> Method:
    return make(cfg["preset"], model, **cfg.get("overrides", {}))


def run_training(config: RunConfig, step_hook=None) -> RunResult:
    """One training run, step times by a monotonic clock around `step` (run.py:213-294)."""
    train, _ = build_dataset(config.dataset)
    model = build_model(config.model)
    method = build_method(config.method, model)
    root = Rng(config.seed)
    init_rng = root.split()
    batch_rng = root.split()
    w = init_params(model, init_rng).to_device()
    state = method.init(w, seed=config.seed)
    batcher = EpochBatcher(train, config.batch_size, batch_rng)
    rows, times = [], []
    for t in range(config.steps):
        batch = batcher.next()
        t0 = time.perf_counter()
        if step_hook is not None:
            step_hook(t)
        w, state, info = method.step(w, batch, state)
        dt = (time.perf_counter() - t0) * 1e3
        times.append(dt)
        rows.append(info.to_row() + [dt])
    return RunResult(rows, timing_summary(times, config.timing.warmup_steps, config.timing.window), w)


# -- cadence study (bench.py:135-207) ---------------------------------------------------
CADENCE_CSV_FIELDS = ("rho_every_k", "median_ms", "p90_ms", "overhead_pct")
PAPER_TABLE3_MS = {-1: (0.84, 0.87), 10: (0.95, 1.16), 5: (0.96, 1.33), 2: (1.30, 1.40), 1: (1.33, 1.34)}


def cadence_methods(ks, model: Model, cg_maxiter: int = 3, cg_warm_start: bool = True) -> dict:
    return {k: make("newton_cg", model, damping={"policy": "constant", "lam0": 1.0, "tr": None},
                    solver={"cg": {"maxiter": cg_maxiter, "warm_start": cg_warm_start}},
                    telemetry={"rho_every_k": k})
            for k in ks}


def bench_cadence(ks=(-1, 10, 5, 2, 1), out_dir=None, steps: int = 1000, width: int = 1024, input_dim: int = 512,
                  batch: int = 256, cg_maxiter: int = 3, cg_warm_start: bool = True, window: int = 50,
                  warmup: int = 2, seed: int = 0, return_infos: bool = False):
    """Steady-state step time of newton_cg as the rho-probe cadence varies (paired).

    Returns rows [rho_every_k, median_ms, p90_ms, overhead_pct] (bench.py:195-202);
    with `return_infos`, also the per-setting StepInfo rows of every step."""
    ks = list(ks)
    train, _ = gen_regression(20000, input_dim, 0.1, 0)
    model = Model(input_dim, (width, width), 1, "relu")
    methods = cadence_methods(ks, model, cg_maxiter, cg_warm_start)
    root = Rng(seed)
    w = init_params(model, root.split()).to_device()
    batcher = EpochBatcher(train, batch, root.split())
    state = methods[ks[0]].init(w, seed=seed)
    times = {k: [] for k in ks}
    infos = {k: [] for k in ks}
    for t in range(steps + warmup):
        b = batcher.next()
        shift = t % len(ks)
        order = ks[shift:] + ks[:shift]
        for k in order:
            t0 = time.perf_counter()
            w_next, state_next, info = methods[k].step(w, b, state)
            times[k].append((time.perf_counter() - t0) * 1e3)
            if return_infos:
                infos[k].append(info.to_row())
        w, state = w_next, state_next
    summaries = {k: timing_summary(times[k], warmup, window) for k in ks}
    base = summaries[-1].median_ms if -1 in summaries else None
    rows = []
    for k in ks:
        med = summaries[k].median_ms
        rows.append([k, med, summaries[k].p90_ms, float("nan") if base is None else (med / base - 1.0) * 100.0])
    if out_dir is not None:
        out = Path(out_dir)
        out.mkdir(parents=True, exist_ok=True)
        with open(out / "cadence.csv", "w", encoding="utf-8") as fh:
            fh.write(",".join(CADENCE_CSV_FIELDS) + "\n")
            for r in rows:
                fh.write(",".join(repr(v) if isinstance(v, float) else str(v) for v in r) + "\n")
        (out / "meta.json").write_text(json.dumps({"study": "cadence", "params": {
            "ks": ks, "steps": steps, "width": width, "batch": batch, "cg_maxiter": cg_maxiter, "seed": seed}},
            indent=2, sort_keys=True))
    return (rows, infos) if return_infos else rows


__all__ = ["Dataset", "DeviceDataset", "EpochBatcher", "gen_regression", "gen_classification", "TimingConfig",
           "RunConfig", "RunResult", "TimingSummary", "timing_summary", "build_dataset", "build_model",
           "build_method", "run_training", "bench_cadence", "cadence_methods", "CADENCE_CSV_FIELDS",
           "PAPER_TABLE3_MS", "STEP_INFO_FIELDS"]
