"""Python front end of the B200 layer-parallel trainer, mirroring the reference's
model/stage/trainer API (include/respar/decoupled.hpp:17-137, network.hpp:29-117)
over the C ABI in include/respar_b200.h.

Arrays cross the boundary as NHWC float32 numpy arrays (host) or raw device pointers
(``*_device`` methods, e.g. ``torch.Tensor.data_ptr()``).  Status codes are re-raised
as the reference's exception types.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import lib, rp_geometry, rp_step_params

SQUARED_L2, L1, LINF = 0, 1, 2          # penalty.hpp:15
SERIAL, PENALTY, ALM = 0, 1, 2          # config.hpp:17
TANH, IDENTITY = 0, 1                   # network.hpp:12
MATH = {"fp32": 0, "tf32": 1, "bf16": 2, "simt": 3}
KAPPA_RULE_REFERENCE, KAPPA_RULE_TEXTBOOK = 0, 1
LAMBDA, KAPPA, BOUNDARY_OUT, BOUNDARY_ADJOINT = 0, 1, 2, 3   # decoupled.hpp:29-32

_PENALTY_NAMES = {"squared_l2": SQUARED_L2, "l1": L1, "linf": LINF}
_MODE_NAMES = {"serial": SERIAL, "penalty": PENALTY, "alm": ALM}


class InvalidArgument(ValueError):
    """std::invalid_argument."""


class ShapeError(InvalidArgument):
    """respar::ShapeError (tensor.hpp:11-13)."""


class ConfigError(InvalidArgument):
    """respar::ConfigError (config.hpp:13-15)."""


class LogicError(RuntimeError):
    """std::logic_error: protocol misuse (decoupled.cpp:89-92, 197-199, 160-163)."""


class StageError(RuntimeError):
    """respar::StageError (runtime.hpp:15-20)."""


class DeviceError(RuntimeError):
    """CUDA / NCCL / internal failure."""


class DivergedError(RuntimeError):
    """std::runtime_error: non-finite loss (decoupled.cpp:249-264)."""


_EXC = {_lib.RP_ERR_SHAPE: ShapeError, _lib.RP_ERR_CONFIG: ConfigError, _lib.RP_ERR_STATE: LogicError,
        _lib.RP_ERR_RANGE: InvalidArgument, _lib.RP_ERR_STAGE: StageError, _lib.RP_ERR_DIVERGED: DivergedError}


def check(rc: int) -> None:
    if rc != 0:
        raise _EXC.get(rc, DeviceError)(f"[rp {rc}] {_lib.last_error()}")


def _kind(v):
    return _PENALTY_NAMES[v] if isinstance(v, str) else int(v)


def _mode(v):
    return _MODE_NAMES[v] if isinstance(v, str) else int(v)


@dataclass
class Geometry:
    """ResidualNet geometry (network.hpp:29-41) + conv geometry."""
    in_channels: int
    height: int
    width: int
    channels: int      # d
    hidden: int        # h
    blocks: int        # L
    classes: int
    activation: int = TANH
    step_h: float = 1.0

    def c(self) -> rp_geometry:
        return rp_geometry(self.in_channels, self.height, self.width, self.channels, self.hidden, self.blocks,
                           self.classes, self.activation, self.step_h)

    @property
    def feature_size(self) -> int:
        return self.height * self.width * self.channels

    @property
    def raw_size(self) -> int:
        return self.height * self.width * self.in_channels


@dataclass
class StepParams:
    """StepParams (decoupled.hpp:45-52) + momentum (0 == reference GD)."""
    beta: float = 1.0
    tau: float = -1.0
    lr: float = 0.1
    lambda_lr: float = 0.1
    kappa_lr: float = 1e-9
    max_corrections: int = 1
    momentum: float = 0.0

    def c(self) -> rp_step_params:
        return rp_step_params(self.beta, self.tau, self.lr, self.lambda_lr, self.kappa_lr, self.max_corrections,
                              self.momentum)


def param_count(g: Geometry) -> int:
    n = lib().rp_param_count(C.byref(g.c()))
    if n < 0:
        raise ConfigError(_lib.last_error())
    return int(n)


def partition(num_blocks: int, stages: int):
    """partition (decoupled.cpp:10-21)."""
    if stages < 1:
        raise ConfigError("partition: need at least one stage")
    if num_blocks < 1 or num_blocks % stages:
        raise ConfigError(f"partition: {stages} stages do not divide {num_blocks} blocks evenly")
    n = num_blocks // stages
    return [(k * n, (k + 1) * n) for k in range(stages)]


def normalizer(nrows: int, feature_size: int) -> int:
    """DecoupledTrainer::normalizer (decoupled.hpp:104-106)."""
    return nrows * feature_size


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


def _ip(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


class DecoupledTrainer:
    """DecoupledTrainer (decoupled.hpp:56-120) running on B200.

    ``params``: flat float32 parameters (include/respar_b200.h layout) or None for the
    device Glorot init from ``seed_state`` (network.cpp:49-68 draw order)."""

    def __init__(self, geometry: Geometry, stages: int, mode, penalty, num_samples: int,
                 params: Optional[np.ndarray] = None, seed_state: int = 0, math: str = "fp32",
                 devices: Optional[Sequence[int]] = None):
        self.geometry = geometry
        self.mode = _mode(mode)
        self.kind = _kind(penalty)
        self.num_samples = num_samples
        self.math = math
        self.nparams = param_count(geometry)
        self._g = geometry.c()
        self._h = C.c_void_p()
        st = C.c_uint64(seed_state)
        p = _f32(params) if params is not None else None
        if p is not None and p.size != self.nparams:
            raise ShapeError(f"params: expected {self.nparams} values, got {p.size}")
        devs = (C.c_int32 * len(devices))(*devices) if devices else None
        check(lib().rp_trainer_create(C.byref(self._g), stages, self.mode, self.kind, num_samples,
                                      _fp(p) if p is not None else None, C.byref(st), MATH[math],
                                      devs, len(devices) if devices else 0, C.byref(self._h)))
        self.seed_state = st.value
        self._stages = stages

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            lib().rp_trainer_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- properties (decoupled.hpp:93-101) ----
    @property
    def stages(self) -> int:
        return self._stages

    @property
    def iteration(self) -> int:
        return int(lib().rp_trainer_iteration(self._h))

    def normalizer(self, nrows: int) -> int:
        return normalizer(nrows, self.geometry.feature_size)

    def set_kappa_rule(self, rule: int) -> None:
        check(lib().rp_trainer_set_kappa_rule(self._h, rule))

    def use_cuda_graphs(self, on: bool = True) -> None:
        """Capture the iteration into a CUDA graph and replay it (rp_trainer_set_graphs)."""
        check(lib().rp_trainer_set_graphs(self._h, 1 if on else 0))

    # ---- parameters ----
    def params(self) -> np.ndarray:
        out = np.empty(self.nparams, np.float32)
        check(lib().rp_trainer_get_params(self._h, _fp(out)))
        return out

    def set_params(self, p) -> None:
        p = _f32(p)
        if p.size != self.nparams:
            raise ShapeError("set_params: size mismatch")
        check(lib().rp_trainer_set_params(self._h, _fp(p)))

    def grads(self) -> np.ndarray:
        out = np.empty(self.nparams, np.float32)
        check(lib().rp_trainer_get_grads(self._h, _fp(out)))
        return out

    # ---- algorithm (decoupled.cpp:44-205) ----
    def _x(self, x, nrows=None):
        x = _f32(x)
        n = x.shape[0] if nrows is None else nrows
        if x.size != n * self.geometry.raw_size:
            raise ShapeError(f"input: expected {n} x {self.geometry.raw_size} values, got {x.size}")
        return x

    def reset_lambda_from_forward(self, full_x) -> None:
        x = _f32(full_x)
        if x.shape[0] != self.num_samples or x.size != self.num_samples * self.geometry.raw_size:
            raise ShapeError("reset_lambda_from_forward: sample count")
        check(lib().rp_trainer_reset_lambda_from_forward(self._h, _fp(x)))

    def step(self, batch_x, labels, row0: int, params: StepParams) -> float:
        x = self._x(batch_x)
        y = np.ascontiguousarray(labels, dtype=np.int32)
        if y.size != x.shape[0]:
            raise ShapeError(f"loss_phi: {y.size} labels for {x.shape[0]} samples")
        loss = C.c_double()
        check(lib().rp_trainer_step(self._h, _fp(x), _ip(y), x.shape[0], row0, C.byref(params.c()), C.byref(loss)))
        return loss.value

    def step_device(self, x_ptr: int, labels_ptr: int, nrows: int, row0: int, params: StepParams,
                    read_loss: bool = False) -> Optional[float]:
        loss = C.c_double()
        check(lib().rp_trainer_step_device(self._h, C.c_void_p(x_ptr), C.c_void_p(labels_ptr), nrows, row0,
                                           C.byref(params.c()), C.byref(loss) if read_loss else None))
        return loss.value if read_loss else None

    def last_loss(self) -> float:
        v = C.c_double()
        check(lib().rp_trainer_last_loss(self._h, C.byref(v)))
        return v.value

    def last_step_ms(self) -> float:
        v = C.c_float()
        check(lib().rp_trainer_last_step_ms(self._h, C.byref(v)))
        return v.value

    def take_snapshot(self, k: int, row0: int, nrows: int) -> None:
        check(lib().rp_trainer_take_snapshot(self._h, k, row0, nrows))

    def stage_forward(self, k: int, batch_x, row0: int, nrows: Optional[int] = None) -> None:
        if k == 0 or batch_x is not None:
            x = self._x(batch_x)
            n = x.shape[0]
            xp = _fp(x)
        else:
            n = nrows
            xp = None
        check(lib().rp_trainer_stage_forward(self._h, k, xp, n, row0))

    def stage_backward_update(self, k: int, labels, beta: float, lr: float, row0: int) -> np.ndarray:
        y = np.ascontiguousarray(labels if labels is not None else [], dtype=np.int32)
        check(lib().rp_trainer_stage_backward_update(self._h, k, _ip(y) if y.size else None, y.size, beta, lr, row0))
        return self.grads()

    def correct_aux(self, k: int, params: StepParams, row0: int, nrows: int) -> None:
        check(lib().rp_trainer_correct_aux(self._h, k, C.byref(params.c()), row0, nrows))

    def correct_multiplier(self, k: int, beta: float, kappa_lr: float, row0: int, nrows: int) -> None:
        check(lib().rp_trainer_correct_multiplier(self._h, k, beta, kappa_lr, row0, nrows))

    def correction_gradient(self, k: int, beta: float, row0: int, nrows: int) -> np.ndarray:
        out = np.empty(nrows * self.geometry.feature_size, np.float32)
        check(lib().rp_trainer_correction_gradient(self._h, k, beta, row0, nrows, _fp(out)))
        return out.reshape(nrows, self.geometry.height, self.geometry.width, self.geometry.channels)

    def violation_report(self):
        per = np.zeros(self.stages)
        mx = C.c_double()
        norm = C.c_int64()
        check(lib().rp_trainer_violation_report(self._h, per.ctypes.data_as(C.POINTER(C.c_double)), C.byref(mx),
                                                C.byref(norm)))
        return list(per), mx.value, norm.value

    # ---- per-stage state (decoupled.hpp:29-32) ----
    def state(self, k: int, which: int) -> np.ndarray:
        g = self.geometry
        if k == 0 and which in (LAMBDA, KAPPA):
            return np.zeros((0, g.height, g.width, g.channels), np.float32)
        out = np.empty((self.num_samples, g.height, g.width, g.channels), np.float32)
        check(lib().rp_trainer_get_state(self._h, k, which, _fp(out)))
        return out

    def set_state(self, k: int, which: int, value) -> None:
        v = _f32(value)
        if v.size != self.num_samples * self.geometry.feature_size:
            raise ShapeError("set_state: size mismatch")
        check(lib().rp_trainer_set_state(self._h, k, which, _fp(v)))

    # ---- evaluation (decoupled.cpp:332-347) ----
    def forward(self, x) -> np.ndarray:
        x = self._x(x)
        out = np.empty((x.shape[0], self.geometry.classes), np.float32)
        check(lib().rp_trainer_forward(self._h, _fp(x), x.shape[0], _fp(out)))
        return out

    def evaluate(self, x, labels):
        """(loss_phi, accuracy) of the current net on (x, labels), computed on device
        (decoupled.cpp:332-347, network.cpp:193-234): the full serial forward, mean softmax-CE,
        argmax hits with ties to the lowest class."""
        x = self._x(x)
        y = np.ascontiguousarray(labels, dtype=np.int32)
        if y.size != x.shape[0]:
            raise ShapeError(f"loss_phi: {y.size} labels for {x.shape[0]} samples")
        loss, acc = C.c_double(), C.c_double()
        check(lib().rp_trainer_evaluate(self._h, _fp(x), _ip(y), x.shape[0], C.byref(loss), C.byref(acc)))
        return loss.value, acc.value

    def accuracy(self, x, labels) -> float:
        """accuracy (network.cpp:223-234): argmax with ties to the lowest class (on device)."""
        return self.evaluate(x, labels)[1]


class SerialTrainer(DecoupledTrainer):
    """The serial baseline (network.cpp:236-244) as the K = 1 path of the same kernels."""

    def __init__(self, geometry: Geometry, num_samples: int, params=None, seed_state: int = 0, math: str = "fp32",
                 devices=None):
        super().__init__(geometry, 1, SERIAL, SQUARED_L2, num_samples, params, seed_state, math, devices)

    def serial_train_step(self, batch, labels, lr: float) -> float:
        x = self._x(batch)
        y = np.ascontiguousarray(labels, dtype=np.int32)
        loss = C.c_double()
        check(lib().rp_serial_train_step(self._h, _fp(x), _ip(y), x.shape[0], lr, C.byref(loss)))
        return loss.value


def serial_train_step(trainer: SerialTrainer, batch, labels, lr: float) -> float:
    """serial_train_step(net, batch, labels, lr) (network.hpp:116-117)."""
    return trainer.serial_train_step(batch, labels, lr)


def launch_count() -> int:
    return int(lib().rp_launch_count())
