"""ctypes binding to oracle/_ref/librespar_ref.so — the *unmodified* reference
library compiled from /root/reference by oracle/build_ref.sh, plus the flat C shim
oracle/ref_shim.cpp.

TEST INFRASTRUCTURE ONLY (golden-vector generation, oracle pinning, and the
reference arm of bench.py).  Never imported by the product package.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "librespar_ref.so")

_D = C.POINTER(C.c_double)
_I = C.POINTER(C.c_int)
_U64 = C.POINTER(C.c_uint64)

_lib = None


class RefError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def available() -> bool:
    return os.path.isfile(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise FileNotFoundError(f"{LIB_PATH} missing: run oracle/build_ref.sh")
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_trainer_create.restype = C.c_void_p
        L.ref_trainer_create.argtypes = [C.c_int] * 6 + [_D] + [C.c_int] * 5
        for name in ("ref_trainer_destroy",):
            getattr(L, name).argtypes = [C.c_void_p]
        L.ref_param_count.restype = C.c_long
        L.ref_trainer_state_size.restype = C.c_long
        L.ref_trainer_state_size.argtypes = [C.c_void_p, C.c_int, C.c_int]
        L.ref_trainer_iteration.restype = C.c_long
        L.ref_trainer_iteration.argtypes = [C.c_void_p]
        L.ref_rng_next_u64.restype = C.c_uint64
        L.ref_rng_split.restype = C.c_uint64
        L.ref_build_initial_net.restype = C.c_int
        for name in ("ref_trainer_get_params", "ref_trainer_set_params", "ref_trainer_reset_lambda",
                     "ref_trainer_get_state", "ref_trainer_set_state", "ref_trainer_step",
                     "ref_trainer_take_snapshot", "ref_trainer_stage_forward",
                     "ref_trainer_stage_backward_update", "ref_trainer_correct_aux",
                     "ref_trainer_correct_multiplier", "ref_trainer_correction_gradient",
                     "ref_trainer_violation_report"):
            getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_D)


def _check(rc):
    if rc != 0:
        raise RefError(rc, lib().ref_last_error().decode())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class RefRng:
    def __init__(self, seed: int):
        self.state = C.c_uint64(seed)

    def uniform(self, rows, cols, lo, hi):
        out = np.empty(rows * cols)
        _check(lib().ref_rng_uniform(C.byref(self.state), rows, cols, C.c_double(lo), C.c_double(hi), _p(out)))
        return out.reshape(rows, cols)

    def normal(self, rows, cols, mean, sigma):
        out = np.empty(rows * cols)
        _check(lib().ref_rng_normal(C.byref(self.state), rows, cols, C.c_double(mean), C.c_double(sigma), _p(out)))
        return out.reshape(rows, cols)

    def next_u64(self):
        return lib().ref_rng_next_u64(C.byref(self.state))

    def split(self):
        r = RefRng(0)
        r.state = C.c_uint64(lib().ref_rng_split(C.byref(self.state)))
        return r


def param_count(in_dim, d, h, L, classes):
    return lib().ref_param_count(in_dim, d, h, L, classes)


def make_net(rng: RefRng, in_dim, d, h, L, classes):
    out = np.empty(param_count(in_dim, d, h, L, classes))
    _check(lib().ref_make_net(C.byref(rng.state), in_dim, d, h, L, classes, _p(out)))
    return out


def serial_train_step(dims, act, params, x, labels, lr):
    in_dim, d, h, L, classes = dims
    params = _f64(params).copy()
    x = _f64(x)
    y = _i32(labels)
    loss = C.c_double()
    _check(lib().ref_serial_train_step(in_dim, d, h, L, classes, act, _p(params), _p(x),
                                       y.ctypes.data_as(_I), x.shape[0], C.c_double(lr), C.byref(loss)))
    return loss.value, params


def net_forward(dims, act, params, x, frm, to):
    in_dim, d, h, L, classes = dims
    x = _f64(x)
    feats = np.empty((x.shape[0], d))
    logits = np.empty((x.shape[0], classes))
    _check(lib().ref_net_forward(in_dim, d, h, L, classes, act, _p(_f64(params)), _p(x), x.shape[0],
                                 frm, to, _p(feats), _p(logits)))
    return feats, logits


def psi(kind, lam, x):
    lam, x = _f64(lam), _f64(x)
    out = C.c_double()
    _check(lib().ref_psi(kind, _p(lam), _p(x), lam.shape[0], lam.shape[1], C.byref(out)))
    return out.value


def psi_grads(kind, lam, x):
    lam, x = _f64(lam), _f64(x)
    dl, dx = np.empty_like(lam), np.empty_like(lam)
    _check(lib().ref_psi_grads(kind, _p(lam), _p(x), lam.shape[0], lam.shape[1], _p(dl), _p(dx)))
    return dl, dx


def loss_phi(logits, labels):
    logits = _f64(logits)
    y = _i32(labels)
    v = C.c_double()
    g = np.empty_like(logits)
    _check(lib().ref_loss_phi(_p(logits), y.ctypes.data_as(_I), logits.shape[0], logits.shape[1],
                              C.byref(v), _p(g)))
    return v.value, g


class RefTrainer:
    """Handle on the reference DecoupledTrainer + StagePool (decoupled.hpp:56)."""

    def __init__(self, dims, act, params, stages, mode, penalty, num_samples, workers=1):
        self.dims = dims
        in_dim, d, h, L, classes = dims
        self.d = d
        self.stages = stages
        self.nparams = param_count(*dims)
        p = _f64(params)
        self.h = lib().ref_trainer_create(in_dim, d, h, L, classes, act, _p(p), stages, mode, penalty,
                                          num_samples, workers)
        if not self.h:
            raise RefError(-1, lib().ref_last_error().decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().ref_trainer_destroy(C.c_void_p(self.h))
            self.h = None

    def params(self):
        out = np.empty(self.nparams)
        _check(lib().ref_trainer_get_params(C.c_void_p(self.h), _p(out)))
        return out

    def set_params(self, p):
        _check(lib().ref_trainer_set_params(C.c_void_p(self.h), _p(_f64(p))))

    def reset_lambda_from_forward(self, x):
        x = _f64(x)
        _check(lib().ref_trainer_reset_lambda(C.c_void_p(self.h), _p(x), x.shape[0], x.shape[1]))

    def state(self, k, which):
        n = lib().ref_trainer_state_size(C.c_void_p(self.h), k, which)
        out = np.empty(n)
        _check(lib().ref_trainer_get_state(C.c_void_p(self.h), k, which, _p(out)))
        return out.reshape(-1, self.d) if n else out

    def set_state(self, k, which, t):
        t = _f64(t)
        _check(lib().ref_trainer_set_state(C.c_void_p(self.h), k, which, _p(t), t.shape[0], t.shape[1]))

    def step(self, x, labels, row0, beta=1.0, tau=-1.0, lr=0.1, lambda_lr=0.1, kappa_lr=1e-9, max_corrections=1):
        x = _f64(x)
        y = _i32(labels)
        loss = C.c_double()
        _check(lib().ref_trainer_step(C.c_void_p(self.h), _p(x), x.shape[0], x.shape[1], y.ctypes.data_as(_I),
                                      row0, C.c_double(beta), C.c_double(tau), C.c_double(lr),
                                      C.c_double(lambda_lr), C.c_double(kappa_lr), max_corrections,
                                      C.byref(loss)))
        return loss.value

    def take_snapshot(self, k, row0, nrows):
        _check(lib().ref_trainer_take_snapshot(C.c_void_p(self.h), k, row0, nrows))

    def stage_forward(self, k, x, row0):
        x = _f64(x)
        _check(lib().ref_trainer_stage_forward(C.c_void_p(self.h), k, _p(x), x.shape[0], x.shape[1], row0))

    def stage_backward_update(self, k, labels, beta, lr, row0, nrows):
        y = _i32(labels) if labels is not None else np.zeros(nrows, np.int32)
        g = np.empty(self.nparams)
        _check(lib().ref_trainer_stage_backward_update(C.c_void_p(self.h), k, y.ctypes.data_as(_I), nrows,
                                                       C.c_double(beta), C.c_double(lr), row0, _p(g)))
        return g

    def correct_aux(self, k, beta, tau, lambda_lr, max_corrections, row0, nrows):
        _check(lib().ref_trainer_correct_aux(C.c_void_p(self.h), k, C.c_double(beta), C.c_double(tau),
                                             C.c_double(lambda_lr), max_corrections, row0, nrows))

    def correct_multiplier(self, k, beta, kappa_lr, row0, nrows):
        _check(lib().ref_trainer_correct_multiplier(C.c_void_p(self.h), k, C.c_double(beta),
                                                    C.c_double(kappa_lr), row0, nrows))

    def correction_gradient(self, k, beta, row0, nrows):
        out = np.empty((nrows, self.d))
        _check(lib().ref_trainer_correction_gradient(C.c_void_p(self.h), k, C.c_double(beta), row0, nrows, _p(out)))
        return out

    def violation_report(self):
        per = np.empty(self.stages)
        mx = C.c_double()
        norm = C.c_long()
        _check(lib().ref_trainer_violation_report(C.c_void_p(self.h), _p(per), C.byref(mx), C.byref(norm)))
        return list(per), mx.value, norm.value


def build_initial_net(mode, init, d, h, L, K, classes, coarse_epochs, warm_epochs, lr_steps, x, labels, state):
    """The reference's build_initial_net (decoupled.cpp:207-245); in_dim is 2 there.
    Returns (flat params, advanced rng state)."""
    Lb = lib()
    n = len(lr_steps)
    ep = (C.c_int * max(n, 1))(*[int(e) for e, _ in lr_steps])
    va = (C.c_double * max(n, 1))(*[float(v) for _, v in lr_steps])
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(labels, np.int32)
    st = C.c_uint64(state)
    out = np.empty(param_count(2, d, h, L, classes), np.float64)
    rc = Lb.ref_build_initial_net(mode, init, d, h, L, K, classes, coarse_epochs, warm_epochs, ep, va, n,
                                  x.ctypes.data_as(_D), y.ctypes.data_as(_I), x.shape[0], C.byref(st),
                                  out.ctypes.data_as(_D))
    if rc != 0:
        raise RefError(rc, Lb.ref_last_error().decode())
    return out, st.value
