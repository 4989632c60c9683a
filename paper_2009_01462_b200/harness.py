"""Experiment harness around the B200 step: the reference's train() loop, configs,
schedules, the toy dataset and the metrics CSV.

Mirrors, name for name, the reference's
  * config.hpp / config.cpp     -- Schedules, TrainConfig, default_schedules, default_config,
                                   parse_config_json, load_config_file (strict keys)
  * dataset.hpp / dataset.cpp   -- Dataset, circles_label, gen_circles
  * metrics.hpp / metrics.cpp   -- MetricsRow, metrics_csv_header, write/read_metrics_csv (%.17g)
  * decoupled.cpp:268-351       -- train(cfg, train_set, test_set): build_initial_net, the epoch
                                   and mini-batch loops with piecewise schedules, the optional
                                   noise on lambda_{K-1}, per-epoch serial-forward evaluation,
                                   the divergence abort
  * experiment.cpp              -- ExperimentSummary, run_experiment, summarize_metrics,
                                   format_summary_table, measure_speedup (runtime.cpp:90-95)

The arithmetic runs on the device trainer (trainer.py over the C ABI); this module is host
control flow only.  The toy problem (2-D points) is the conv geometry with H = W = 1 and
Cin = 2, on which the B200 net *is* the reference's dense ResidualNet.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import time
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import init as _init
from ._lib import lib
from .trainer import (ALM, LAMBDA, PENALTY, SQUARED_L2, ConfigError, DecoupledTrainer, DivergedError, Geometry,
                      SerialTrainer, StepParams, check)

Steps = List[Tuple[int, float]]

_MASK = (1 << 64) - 1
_GAMMA = 0x9E3779B97F4A7C15


class Rng:
    """splitmix64 Rng (tensor.cpp:163-175), bit-identical to the reference."""

    def __init__(self, seed: int):
        self.state = seed & _MASK

    def next_u64(self) -> int:
        self.state = (self.state + _GAMMA) & _MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK
        return z ^ (z >> 31)

    def next_double(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def split(self) -> "Rng":
        return Rng(self.next_u64())


# ------------------------------------------------------------------ config
@dataclass
class Schedules:
    """Schedules (config.hpp:28-43)."""
    beta_steps: Steps = field(default_factory=list)
    tau_steps: Steps = field(default_factory=list)
    lr_steps: Steps = field(default_factory=list)
    lambda_lr_steps: Steps = field(default_factory=list)
    lambda_lr_scale: float = 1.0
    kappa_lr: float = 1e-9
    correction_max_iters: int = 1
    noise_sigma_last: float = 0.0

    @staticmethod
    def value_at(steps: Sequence[Tuple[int, float]], epoch: int, fallback: float) -> float:
        return _init.lr_value_at(steps, epoch, fallback)

    def validate(self) -> None:
        """Schedules::validate (config.cpp:54-62)."""
        def steps_ok(name, steps, positive):
            prev = -1
            for e, v in steps:
                if e < 0:
                    raise ConfigError(f"{name}: negative epoch")
                if e <= prev:
                    raise ConfigError(f"{name}: epochs must be strictly increasing")
                if positive and v <= 0.0:
                    raise ConfigError(f"{name}: values must be positive")
                prev = e
        steps_ok("beta schedule", self.beta_steps, True)
        steps_ok("tau schedule", self.tau_steps, False)
        steps_ok("lr schedule", self.lr_steps, True)
        steps_ok("lambda_lr schedule", self.lambda_lr_steps, True)
        if self.lambda_lr_scale < 0.0:
            raise ConfigError("lambda_lr_scale must be >= 0")
        if self.kappa_lr < 0.0:
            raise ConfigError("kappa_lr must be >= 0")
        if self.correction_max_iters < 1:
            raise ConfigError("correction_max_iters must be >= 1")
        if self.noise_sigma_last < 0.0:
            raise ConfigError("noise_sigma_last must be >= 0")


@dataclass
class TrainConfig:
    """TrainConfig (config.hpp:46-68) + the conv geometry of the B200 build (the
    reference's toy problem is in_channels 2, height = width = 1)."""
    mode: str = "serial"
    stages: int = 1
    num_blocks: int = 60
    feature_dim: int = 8
    hidden_dim: int = 8
    classes: int = 3
    epochs: int = 300
    batch_size: int = 0
    seed: int = 0
    train_points: int = 200
    test_points: int = 200
    penalty: str = "squared_l2"
    schedules: Schedules = field(default_factory=Schedules)
    init: str = "multilevel"
    coarse_epochs: int = 50
    warmstart_epochs: int = 10
    workers: int = 0
    out_path: str = ""
    emit_timing: bool = True
    in_channels: int = 2
    height: int = 1
    width: int = 1
    math: str = "fp32"

    def validate(self) -> None:
        """TrainConfig::validate (config.cpp:82-99)."""
        if self.mode not in ("serial", "penalty", "alm"):
            raise ConfigError(f"unknown mode '{self.mode}' (expected serial, penalty or alm)")
        if self.stages < 1:
            raise ConfigError("stages must be >= 1")
        if self.num_blocks < 1:
            raise ConfigError("blocks must be >= 1")
        if self.num_blocks % self.stages != 0:
            raise ConfigError(f"stage count {self.stages} does not divide {self.num_blocks} blocks")
        if self.feature_dim < 1 or self.hidden_dim < 1:
            raise ConfigError("widths must be >= 1")
        if self.classes < 2:
            raise ConfigError("classes must be >= 2")
        if self.epochs < 1:
            raise ConfigError("epochs must be >= 1")
        if self.batch_size < 0:
            raise ConfigError("batch_size must be >= 0")
        if self.train_points < 1 or self.test_points < 1:
            raise ConfigError("dataset sizes must be >= 1")
        if self.mode == "serial" and self.stages != 1:
            raise ConfigError("serial mode runs exactly one stage")
        if self.init not in ("multilevel", "warmstart", "random"):
            raise ConfigError(f"unknown init scheme '{self.init}' (expected multilevel, warmstart or random)")
        if self.penalty not in ("squared_l2", "l1", "linf"):
            raise ConfigError(f"unknown penalty '{self.penalty}'")
        self.schedules.validate()

    def geometry(self) -> Geometry:
        return Geometry(self.in_channels, self.height, self.width, self.feature_dim, self.hidden_dim,
                        self.num_blocks, self.classes)


def default_schedules(mode: str) -> Schedules:
    """default_schedules (config.cpp:102-111): lr 0.1 cut 10x at epochs 70 / 150; beta 1
    (penalty) or 0.1 (ALM) raised 10x at 100 / 250."""
    s = Schedules(lr_steps=[(0, 0.1), (70, 0.01), (150, 0.001)])
    s.beta_steps = [(0, 0.1), (100, 1.0), (250, 10.0)] if mode == "alm" else [(0, 1.0), (100, 10.0), (250, 100.0)]
    return s


def default_config(mode: str) -> TrainConfig:
    """default_config (config.cpp:113-119)."""
    return TrainConfig(mode=mode, stages=1 if mode == "serial" else 2, schedules=default_schedules(mode))


_CONFIG_KEYS = {"mode", "stages", "blocks", "feature_dim", "hidden_dim", "classes", "epochs", "batch_size", "seed",
                "train_points", "test_points", "penalty", "schedules", "init", "coarse_epochs", "warmstart_epochs",
                "workers", "out", "emit_timing"}
_SCHED_KEYS = {"beta", "tau", "lr", "lambda_lr", "lambda_lr_scale", "kappa_lr", "correction_max_iters",
               "noise_sigma_last"}


def _steps(v, key) -> Steps:
    if not isinstance(v, list):
        raise ConfigError(f"{key}: expected an array of [epoch, value] pairs")
    out = []
    for item in v:
        if (not isinstance(item, list) or len(item) != 2 or not isinstance(item[0], int) or isinstance(item[0], bool)
                or not isinstance(item[1], (int, float)) or isinstance(item[1], bool)):
            raise ConfigError(f"{key}: expected [epoch, value] pairs")
        out.append((int(item[0]), float(item[1])))
    return out


def _typed(v, types, key):
    if isinstance(v, bool) and bool not in types:
        raise ConfigError(f"config type error: {key}")
    if not isinstance(v, types):
        raise ConfigError(f"config type error: {key}")
    return v


def parse_config_json(text: str, base: Optional[TrainConfig] = None) -> TrainConfig:
    """parse_config_json (config.cpp:160-206): strict keys, type errors -> ConfigError."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise ConfigError(f"config parse error: {e}") from e
    if not isinstance(j, dict):
        raise ConfigError("config root must be an object")
    for k in j:
        if k not in _CONFIG_KEYS:
            raise ConfigError(f"config: unknown key '{k}'")
    import copy
    cfg = copy.deepcopy(base) if base is not None else TrainConfig()
    if "mode" in j:
        cfg.mode = _typed(j["mode"], (str,), "mode")
        if cfg.mode not in ("serial", "penalty", "alm"):
            raise ConfigError(f"unknown mode '{cfg.mode}' (expected serial, penalty or alm)")
        cfg.schedules = default_schedules(cfg.mode)     # a mode change re-bases the schedules
    ints = {"stages": "stages", "blocks": "num_blocks", "feature_dim": "feature_dim", "hidden_dim": "hidden_dim",
            "classes": "classes", "epochs": "epochs", "batch_size": "batch_size", "seed": "seed",
            "train_points": "train_points", "test_points": "test_points", "coarse_epochs": "coarse_epochs",
            "warmstart_epochs": "warmstart_epochs", "workers": "workers"}
    for k, attr in ints.items():
        if k in j:
            setattr(cfg, attr, _typed(j[k], (int,), k))
    if "penalty" in j:
        cfg.penalty = _typed(j["penalty"], (str,), "penalty")
    if "init" in j:
        cfg.init = _typed(j["init"], (str,), "init")
    if "out" in j:
        cfg.out_path = _typed(j["out"], (str,), "out")
    if "emit_timing" in j:
        cfg.emit_timing = _typed(j["emit_timing"], (bool,), "emit_timing")
    if "schedules" in j:
        sj = j["schedules"]
        if not isinstance(sj, dict):
            raise ConfigError("config type error: schedules")
        for k in sj:
            if k not in _SCHED_KEYS:
                raise ConfigError(f"schedules: unknown key '{k}'")
        s = cfg.schedules
        if "beta" in sj:
            s.beta_steps = _steps(sj["beta"], "schedules.beta")
        if "tau" in sj:
            s.tau_steps = _steps(sj["tau"], "schedules.tau")
        if "lr" in sj:
            s.lr_steps = _steps(sj["lr"], "schedules.lr")
        if "lambda_lr" in sj:
            s.lambda_lr_steps = _steps(sj["lambda_lr"], "schedules.lambda_lr")
        if "lambda_lr_scale" in sj:
            s.lambda_lr_scale = float(_typed(sj["lambda_lr_scale"], (int, float), "lambda_lr_scale"))
        if "kappa_lr" in sj:
            s.kappa_lr = float(_typed(sj["kappa_lr"], (int, float), "kappa_lr"))
        if "correction_max_iters" in sj:
            s.correction_max_iters = _typed(sj["correction_max_iters"], (int,), "correction_max_iters")
        if "noise_sigma_last" in sj:
            s.noise_sigma_last = float(_typed(sj["noise_sigma_last"], (int, float), "noise_sigma_last"))
    cfg.validate()
    return cfg


def load_config_file(path: str, base: Optional[TrainConfig] = None) -> TrainConfig:
    """load_config_file (config.cpp:208-215)."""
    try:
        with open(path) as f:
            text = f.read()
    except OSError as e:
        raise ConfigError(f"cannot read config '{path}'") from e
    return parse_config_json(text, base)


# ------------------------------------------------------------------ dataset
@dataclass
class Dataset:
    """Dataset (dataset.hpp:14-17): points as NHWC [n, 1, 1, 2] float32."""
    points: np.ndarray
    labels: np.ndarray


def circles_label(x: float, y: float) -> int:
    """circles_label (dataset.cpp:10-15): points exactly on a circle go inward."""
    r = math.hypot(x, y)
    if r <= 0.5:
        return 0
    if r <= 0.75:
        return 1
    return 2


def gen_circles(n: int, seed: int) -> Dataset:
    """gen_circles (dataset.cpp:17-26): rng_uniform(n, 2, -1, 1), then labels."""
    if n < 1:
        raise ValueError("gen_circles: n must be >= 1")
    rng = Rng(seed)
    pts = np.array([-1.0 + 2.0 * rng.next_double() for _ in range(2 * n)]).reshape(n, 2)
    labels = np.array([circles_label(pts[i, 0], pts[i, 1]) for i in range(n)], np.int32)
    return Dataset(points=pts.reshape(n, 1, 1, 2).astype(np.float32), labels=labels)


# ------------------------------------------------------------------ metrics
@dataclass
class MetricsRow:
    """MetricsRow (metrics.hpp:11-21)."""
    epoch: int = 0
    train_loss: float = 0.0
    test_accuracy: float = 0.0
    max_violation: float = 0.0
    beta: float = 0.0
    lr: float = 0.0
    epoch_seconds: float = 0.0


def metrics_csv_header() -> str:
    return "epoch,train_loss,test_accuracy,max_violation,beta,lr,epoch_seconds"


def write_metrics_csv(rows: Sequence[MetricsRow], path: str) -> None:
    """write_metrics_csv (metrics.cpp:15-27): %.17g."""
    with open(path, "w") as f:
        f.write(metrics_csv_header() + "\n")
        for r in rows:
            f.write("%d,%.17g,%.17g,%.17g,%.17g,%.17g,%.17g\n" % (r.epoch, r.train_loss, r.test_accuracy,
                                                                    r.max_violation, r.beta, r.lr, r.epoch_seconds))


def read_metrics_csv(path: str) -> List[MetricsRow]:
    """read_metrics_csv (metrics.cpp:29-56)."""
    with open(path) as f:
        lines = f.read().split("\n")
    if not lines or lines[0] != metrics_csv_header():
        raise RuntimeError(f"'{path}' is not a metrics file (bad header)")
    rows = []
    for ln in lines[1:]:
        if not ln:
            continue
        parts = ln.split(",")
        if len(parts) < 7:
            raise RuntimeError(f"'{path}': short row '{ln}'")
        try:
            v = [float(p) for p in parts[:7]]
        except ValueError as e:
            raise RuntimeError(f"'{path}': bad number in '{ln}'") from e
        rows.append(MetricsRow(int(v[0]), *v[1:]))
    return rows


# ------------------------------------------------------------------ train
@dataclass
class EpochTiming:
    epoch: int = 0
    train_wall_seconds: float = 0.0


@dataclass
class TrainResult:
    """TrainResult (decoupled.hpp:128-133); `params` is the trained flat parameters."""
    metrics: List[MetricsRow] = field(default_factory=list)
    timings: List[EpochTiming] = field(default_factory=list)
    init_seconds: float = 0.0
    params: Optional[np.ndarray] = None


def train(cfg: TrainConfig, train_set: Dataset, test_set: Dataset) -> TrainResult:
    """train (decoupled.cpp:268-351) on the B200 trainer."""
    cfg.validate()
    g = cfg.geometry()
    n_train = train_set.points.shape[0]
    batch = n_train if cfg.batch_size == 0 else min(cfg.batch_size, n_train)
    root = Rng(cfg.seed)
    net_rng = root.split()
    noise_rng = root.split()
    res = TrainResult()
    t_init = time.perf_counter()
    params, _ = _init.build_initial_net(
        g, cfg.stages, cfg.mode, cfg.init, train_set.points, train_set.labels, net_rng.state,
        coarse_epochs=cfg.coarse_epochs, warmstart_epochs=cfg.warmstart_epochs, lr_steps=cfg.schedules.lr_steps,
        math=cfg.math)
    if cfg.mode == "serial":
        tr = SerialTrainer(g, batch, params=params, math=cfg.math)
    else:
        tr = DecoupledTrainer(g, cfg.stages, ALM if cfg.mode == "alm" else PENALTY, cfg.penalty, n_train,
                              params=params, math=cfg.math)
        tr.reset_lambda_from_forward(train_set.points)
    res.init_seconds = time.perf_counter() - t_init
    sch = cfg.schedules
    noise_state = C.c_uint64(noise_rng.state)
    last = cfg.stages - 1
    for epoch in range(cfg.epochs):
        sp = StepParams(beta=sch.value_at(sch.beta_steps, epoch, 1.0), tau=sch.value_at(sch.tau_steps, epoch, -1.0),
                        lr=sch.value_at(sch.lr_steps, epoch, 0.1), kappa_lr=sch.kappa_lr,
                        max_corrections=sch.correction_max_iters)
        sp.lambda_lr = (sp.lr * sch.lambda_lr_scale if not sch.lambda_lr_steps
                        else sch.value_at(sch.lambda_lr_steps, epoch, sp.lr))
        t0 = time.perf_counter()
        for row0 in range(0, n_train, batch):
            nrows = min(batch, n_train - row0)
            xb = train_set.points[row0:row0 + nrows]
            yb = train_set.labels[row0:row0 + nrows]
            if cfg.mode == "serial":
                tr.serial_train_step(xb, yb, sp.lr)
            else:
                tr.step(xb, yb, row0, sp)
                if sch.noise_sigma_last > 0.0 and cfg.stages >= 2:
                    # lambda_{K-1} rows += N(0, sigma^2) from the noise stream (decoupled.cpp:315-321)
                    ptr = C.c_void_p()
                    check(lib().rp_trainer_state_device(tr._h, last, LAMBDA, C.byref(ptr)))
                    s = C.c_void_p()
                    check(lib().rp_trainer_stage_stream(tr._h, last, C.byref(s)))
                    fs = g.feature_size
                    check(lib().rp_op_fill_normal(C.c_void_p(ptr.value + 4 * row0 * fs), nrows * fs,
                                                  C.byref(noise_state), 0.0, sch.noise_sigma_last, 1, s))
        wall = time.perf_counter() - t0
        res.timings.append(EpochTiming(epoch, wall))
        # evaluation through a full serial forward pass; excluded from timings
        train_loss, _ = tr.evaluate(train_set.points, train_set.labels)   # on device
        if not math.isfinite(train_loss):
            raise DivergedError(f"training diverged: non-finite loss at epoch {epoch} (mode {cfg.mode}, "
                                f"K={cfg.stages})")
        _, test_acc = tr.evaluate(test_set.points, test_set.labels)
        row = MetricsRow(epoch=epoch, train_loss=train_loss, test_accuracy=test_acc, lr=sp.lr,
                         epoch_seconds=wall if cfg.emit_timing else 0.0)
        if cfg.mode != "serial":
            row.max_violation = tr.violation_report()[1]
            row.beta = sp.beta
        res.metrics.append(row)
    res.params = tr.params()
    return res


# ------------------------------------------------------------------ experiment
@dataclass
class ExperimentSummary:
    """ExperimentSummary (experiment.hpp:12-19)."""
    final_train_loss: float = 0.0
    final_test_accuracy: float = 0.0
    train_wall_seconds: float = 0.0
    mean_epoch_seconds: float = 0.0
    init_seconds: float = 0.0
    speedup: float = 0.0


@dataclass
class ExperimentResult:
    summary: ExperimentSummary
    metrics: List[MetricsRow]


def measure_speedup(serial_wall_seconds: float, parallel_wall_seconds: float) -> float:
    """measure_speedup (runtime.cpp:90-95)."""
    if serial_wall_seconds <= 0.0 or parallel_wall_seconds <= 0.0:
        raise ValueError("measure_speedup: durations must be positive")
    return serial_wall_seconds / parallel_wall_seconds


def run_experiment(cfg: TrainConfig, serial_ref_path: str = "") -> ExperimentResult:
    """run_experiment (experiment.cpp:20-42): circles data (seed, seed + 1), train, summary."""
    cfg.validate()
    trained = train(cfg, gen_circles(cfg.train_points, cfg.seed), gen_circles(cfg.test_points, cfg.seed + 1))
    s = ExperimentSummary(final_train_loss=trained.metrics[-1].train_loss,
                          final_test_accuracy=trained.metrics[-1].test_accuracy,
                          train_wall_seconds=sum(t.train_wall_seconds for t in trained.timings),
                          init_seconds=trained.init_seconds)
    s.mean_epoch_seconds = s.train_wall_seconds / len(trained.timings)
    if serial_ref_path:
        s.speedup = measure_speedup(sum(r.epoch_seconds for r in read_metrics_csv(serial_ref_path)),
                                    s.train_wall_seconds)
    if cfg.out_path:
        write_metrics_csv(trained.metrics, cfg.out_path)
    return ExperimentResult(summary=s, metrics=trained.metrics)


def summarize_metrics(rows: Sequence[MetricsRow], serial_ref_path: str = "") -> ExperimentSummary:
    """summarize_metrics (experiment.cpp:44-57)."""
    if not rows:
        raise ValueError("summarize_metrics: no rows")
    s = ExperimentSummary(final_train_loss=rows[-1].train_loss, final_test_accuracy=rows[-1].test_accuracy,
                          train_wall_seconds=sum(r.epoch_seconds for r in rows))
    s.mean_epoch_seconds = s.train_wall_seconds / len(rows)
    if serial_ref_path:
        s.speedup = measure_speedup(sum(r.epoch_seconds for r in read_metrics_csv(serial_ref_path)),
                                    s.train_wall_seconds)
    return s


def format_summary_table(summary: ExperimentSummary) -> str:
    """format_summary_table (experiment.cpp:59-71)."""
    out = "train loss   test acc.   runtime    speedup\n"
    if summary.speedup > 0.0:
        return out + "%-12.3g %-11.1f%% %-10.2fs %.2f\n" % (summary.final_train_loss,
                                                          100.0 * summary.final_test_accuracy,
                                                          summary.train_wall_seconds, summary.speedup)
    return out + "%-12.3g %-11.1f%% %-10.2fs -\n" % (summary.final_train_loss, 100.0 * summary.final_test_accuracy,
                                                    summary.train_wall_seconds)


__all__ = ["Rng", "Schedules", "TrainConfig", "default_schedules", "default_config", "parse_config_json",
           "load_config_file", "Dataset", "circles_label", "gen_circles", "MetricsRow", "metrics_csv_header",
           "write_metrics_csv", "read_metrics_csv", "TrainResult", "train", "ExperimentSummary", "ExperimentResult",
           "measure_speedup", "run_experiment", "summarize_metrics", "format_summary_table", "SQUARED_L2"]
