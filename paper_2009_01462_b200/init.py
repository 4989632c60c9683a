"""Initialisation of the deep net (build_initial_net, decoupled.cpp:207-245) on B200.

* ``random``     -- the device Glorot init in make_net order (network.cpp:49-68);
* ``warmstart``  -- ``warmstart_epochs`` full-batch serial steps of the deep net;
* ``multilevel`` -- the paper's init (the reference default, config.hpp:60): train the
  K-block coarse net for ``coarse_epochs`` full-batch serial steps, then copy coarse
  block k into the n = L / K blocks of stage k with W2, b2 scaled by 1 / n, so the deep
  net starts out computing (nearly) the trained coarse map.

The serial steps run on the same tcgen05 kernels as the training step (the K = 1 path,
``SerialTrainer``); the replication is a host-side relayout of the flat parameters.
"""
from __future__ import annotations

from dataclasses import replace
from typing import Sequence, Tuple

import numpy as np

from .trainer import ConfigError, Geometry, SerialTrainer, param_count

MULTILEVEL, WARMSTART, RANDOM = "multilevel", "warmstart", "random"   # init_scheme_name (config.cpp)


def lr_value_at(steps: Sequence[Tuple[int, float]], epoch: int, fallback: float = 0.1) -> float:
    """Schedules::value_at (config.cpp:72-80)."""
    v = fallback
    for e, val in steps:
        if e > epoch:
            break
        v = val
    return v


def _block_slices(g: Geometry):
    """Offsets of (s.w, s.b), the L blocks (w1, b1, w2, b2) and (t.w, t.b) in the flat layout."""
    C, Ch, Cin = g.channels, g.hidden, g.in_channels
    s = 9 * Cin * C + C
    blk = [9 * C * Ch, Ch, 9 * Ch * C, C]
    bs = sum(blk)
    return s, blk, bs


def replicate_coarse(g: Geometry, stages: int, coarse_flat: np.ndarray) -> np.ndarray:
    """decoupled.cpp:228-244 on flat parameter vectors."""
    if g.blocks % stages != 0:
        raise ConfigError(f"multilevel init: {stages} stages do not divide {g.blocks} blocks")
    n = g.blocks // stages
    s, blk, bs = _block_slices(g)
    out = np.empty(param_count(g), np.float32)
    out[:s] = coarse_flat[:s]
    for k in range(stages):
        cb = coarse_flat[s + k * bs: s + (k + 1) * bs].copy()
        w2_0 = blk[0] + blk[1]
        cb[w2_0:] *= np.float32(1.0 / n)                      # w2 and b2
        for i in range(n):
            l = k * n + i
            out[s + l * bs: s + (l + 1) * bs] = cb
    out[s + g.blocks * bs:] = coarse_flat[s + stages * bs:]
    return out


def build_initial_net(g: Geometry, stages: int, mode: str, init: str, train_x: np.ndarray, labels: np.ndarray,
                      seed_state: int, coarse_epochs: int = 50, warmstart_epochs: int = 10,
                      lr_steps: Sequence[Tuple[int, float]] = (), math: str = "fp32") -> Tuple[np.ndarray, int]:
    """build_initial_net(cfg, train_x, labels, rng) (decoupled.hpp:125).  Returns the
    flat fp32 parameters of the L-block net and the advanced rng state."""
    lr_at = lambda e: lr_value_at(lr_steps, e, 0.1)  # noqa: E731
    x = np.ascontiguousarray(train_x, np.float32)
    y = np.ascontiguousarray(labels, np.int32)
    rows = x.shape[0]
    if mode == "serial" or init == RANDOM:
        tr = SerialTrainer(g, max(rows, 1), seed_state=seed_state, math=math)
        return tr.params(), tr.seed_state
    if init == WARMSTART:
        tr = SerialTrainer(g, rows, seed_state=seed_state, math=math)
        for e in range(warmstart_epochs):
            tr.serial_train_step(x, y, lr_at(e))
        return tr.params(), tr.seed_state
    if init != MULTILEVEL:
        raise ConfigError(f"unknown init scheme '{init}'")
    cg = replace(g, blocks=stages)
    tr = SerialTrainer(cg, rows, seed_state=seed_state, math=math)
    for e in range(coarse_epochs):
        tr.serial_train_step(x, y, lr_at(e))
    return replicate_coarse(g, stages, tr.params()), tr.seed_state
