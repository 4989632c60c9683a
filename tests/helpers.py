"""Shared test helpers: golden fixtures, geometry embedding, tolerances."""
from __future__ import annotations

import os

import numpy as np

from oracle import respar_oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")

# fp32 device arithmetic vs the fp64 reference/oracle: max-norm relative tolerance
# (north_star: "for example 1e-4 relative after one iteration").
FP32_TOL = 1e-4


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name + ".npz")))


def dense_geometry(dims, act=O.TANH):
    """Reference dims (in_dim, d, h, L, classes) as the conv geometry at H = W = 1."""
    in_dim, d, h, L, classes = (int(v) for v in dims)
    return O.Geometry(in_channels=in_dim, height=1, width=1, channels=d, hidden=h, blocks=L, classes=classes,
                      activation=act)


def rel_err(got, want):
    """max |got - want| / max(|want|_inf, tiny): the per-tensor max-norm relative error."""
    got = np.asarray(got, np.float64).reshape(-1)
    want = np.asarray(want, np.float64).reshape(-1)
    if want.size == 0:
        return 0.0
    scale = max(np.abs(want).max(), 1e-30)
    return float(np.abs(got - want).max() / scale)


def split_params(g: O.Geometry, flat):
    """Flat parameter vector -> list of (name, array) in the reference draw order."""
    net = O.zero_net(g)
    net.load_flat(np.asarray(flat, np.float64))
    out = [("s.w", net.s_w), ("s.b", net.s_b)]
    for l in range(g.blocks):
        out += [(f"b{l}.w1", net.w1[l]), (f"b{l}.b1", net.b1[l]), (f"b{l}.w2", net.w2[l]), (f"b{l}.b2", net.b2[l])]
    return out + [("t.w", net.t_w), ("t.b", net.t_b)]


def param_rel_errs(g, got, want):
    return {n: rel_err(a, b) for (n, a), (_, b) in zip(split_params(g, got), split_params(g, want))}
