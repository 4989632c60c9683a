"""Generates the golden fixtures in tests/golden/*.npz from the REFERENCE itself
(oracle/_ref/librespar_ref.so, compiled from /root/reference/proj/src by
oracle/build_ref.sh).  Run here (the reference is not on the GPU box):

    bash oracle/build_ref.sh && python tests/golden/make_golden.py

Every instance is the reference ResidualNet/DecoupledTrainer on rows = samples, which
is exactly the conv net at H = W = 1 (centre taps).  Initial parameters and inputs
are rounded to fp32 before they enter the reference, so an fp32 device run starts
from bit-identical values.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import refbind as R  # noqa: E402


def f32(a):
    return np.asarray(a, np.float32).astype(np.float64)


def trainer_run(name, dims, K, mode, penalty, N, batch, epochs, sp, seed, kappa_init=None, noise=None,
                lam_perturb=None):
    in_dim, d, h, L, classes = dims
    rng = R.RefRng(seed)
    params = f32(R.make_net(rng, *dims))
    x = f32(rng.uniform(N, in_dim, -1.0, 1.0))
    y = np.array([rng.next_u64() % classes for _ in range(N)], np.int32)
    tr = R.RefTrainer(dims, 0, params, K, mode, penalty, N, workers=1)
    tr.reset_lambda_from_forward(x)
    if kappa_init is not None:
        krng = R.RefRng(kappa_init)
        for k in range(1, K):
            tr.set_state(k, 1, f32(krng.uniform(N, d, -0.05, 0.05)))
    if lam_perturb is not None:
        # lambda_k off the forward states: every stage's synthetic loss is non-stationary, so
        # stage 0's gradients are non-zero from the first step
        prng = R.RefRng(seed + 1000)
        for k in range(1, K):
            tr.set_state(k, 0, f32(tr.state(k, 0) + prng.uniform(N, d, -lam_perturb, lam_perturb)))
    kappa0 = [tr.state(k, 1) for k in range(1, K)]
    lam0 = [tr.state(k, 0) for k in range(1, K)]
    losses = []
    for _ in range(epochs):
        for r0 in range(0, N, batch):
            nr = min(batch, N - r0)
            losses.append(tr.step(x[r0:r0 + nr], y[r0:r0 + nr], r0, **sp))
    out = dict(dims=np.array(dims), K=K, mode=mode, penalty=penalty, N=N, batch=batch, epochs=epochs,
               params0=params, x=x, y=y, losses=np.array(losses), params=tr.params(),
               sp=np.array([sp["beta"], sp["tau"], sp["lr"], sp["lambda_lr"], sp["kappa_lr"],
                            sp["max_corrections"]]))
    for k in range(1, K):
        out[f"kappa0_{k}"] = kappa0[k - 1]
        if lam_perturb is not None:
            out[f"lam0_{k}"] = lam0[k - 1]
    for k in range(K):
        for w, nm in enumerate(("lam", "kappa", "bout", "badj")):
            v = tr.state(k, w)
            if v.size:
                out[f"{nm}_{k}"] = v
    per, mx, norm = tr.violation_report()
    out["violation"] = np.array(per)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "losses", out["losses"][:3], "...", "viol", mx)


def pieces(name, seed=7, dims=(3, 6, 5, 6, 4), K=3, N=9):
    """stage_backward_update gradients for every stage under a frozen snapshot, the
    correction gradient, and one correct_aux / correct_multiplier (decoupled.cpp:65-170)."""
    in_dim, d, h, L, classes = dims
    rng = R.RefRng(seed)
    params = f32(R.make_net(rng, *dims))
    x = f32(rng.uniform(N, in_dim, -1.0, 1.0))
    y = np.array([rng.next_u64() % classes for _ in range(N)], np.int32)
    tr = R.RefTrainer(dims, 0, params, K, 2, 0, N)
    tr.reset_lambda_from_forward(x)
    lam = {}
    kap = {}
    for k in range(1, K):
        lam[k] = f32(tr.state(k, 0) + rng.uniform(N, d, -0.1, 0.1))
        kap[k] = f32(rng.uniform(N, d, -0.05, 0.05))
        tr.set_state(k, 0, lam[k])
        tr.set_state(k, 1, kap[k])
    beta, lr = 1.7, 0.05
    out = dict(dims=np.array(dims), K=K, N=N, params0=params, x=x, y=y, beta=beta, lr=lr)
    for k in range(1, K):
        out[f"lam_in_{k}"] = lam[k]
        out[f"kappa_in_{k}"] = kap[k]
    for k in range(K):
        if k + 1 < K:
            tr.take_snapshot(k, 0, N)
        tr.stage_forward(k, x, 0)
        out[f"bout_{k}"] = tr.state(k, 2)
        out[f"grads_{k}"] = tr.stage_backward_update(k, y if k == K - 1 else None, beta, lr, 0, N)
        out[f"badj_{k}"] = tr.state(k, 3)
    out["params1"] = tr.params()
    for k in range(1, K):
        out[f"corrgrad_{k}"] = tr.correction_gradient(k, beta, 0, N)
        tr.correct_aux(k, beta, -1.0, 0.3, 1, 0, N)
        out[f"lam_corr_{k}"] = tr.state(k, 0)
        tr.correct_multiplier(k, beta, 1e-3, 0, N)
        out[f"kappa_corr_{k}"] = tr.state(k, 1)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, "ok")


def serial(name, seed=6):
    dims = (2, 4, 4, 6, 3)
    rng = R.RefRng(seed)
    params = f32(R.make_net(rng, *dims))
    x = f32(rng.uniform(10, 2, -1.0, 1.0))
    y = np.array([rng.next_u64() % 3 for _ in range(10)], np.int32)
    p = params.copy()
    losses = []
    for _ in range(5):
        loss, p = R.serial_train_step(dims, 0, p, x, y, 0.05)
        losses.append(loss)
    np.savez_compressed(os.path.join(HERE, name + ".npz"), dims=np.array(dims), params0=params, x=x, y=y,
                        losses=np.array(losses), params=p, lr=0.05)
    print(name, losses)


def psi_kats(name):
    """penalty.cpp KATs (test_penalty.cpp:32-38, 61-82, 130-142) + random cases."""
    out = {}
    lam = np.array([[1.0, 2.0]])
    x = np.zeros((1, 2))
    for kind in range(3):
        out[f"kat_psi_{kind}"] = R.psi(kind, lam, x)
        out[f"kat_dl_{kind}"] = R.psi_grads(kind, lam, x)[0]
    rng = R.RefRng(3)
    a = f32(rng.uniform(7, 5, -1, 1))
    b = f32(rng.uniform(7, 5, -1, 1))
    b[2, 3] = a[2, 3]                 # a zero difference (sign0(0) == 0)
    a[4, 1], b[4, 1] = 0.95, -0.95    # exact |d| tie for LInf (fp32 and fp64): first index wins
    a[5, 2], b[5, 2] = -0.95, 0.95
    a, b = f32(a), f32(b)
    assert np.argmax(np.abs(a - b)) == 4 * 5 + 1
    out["a"], out["b"] = a, b
    for kind in range(3):
        out[f"psi_{kind}"] = R.psi(kind, a, b)
        out[f"dl_{kind}"] = R.psi_grads(kind, a, b)[0]
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(name, [out[f"psi_{k}"] for k in range(3)])


if __name__ == "__main__":
    trainer_run("ref_k2_penalty", (3, 8, 6, 4, 5), 2, 1, 0, 12, 12, 3,
                dict(beta=1.0, tau=-1.0, lr=0.05, lambda_lr=0.05, kappa_lr=1e-9, max_corrections=1), seed=11)
    trainer_run("ref_k4_alm_minibatch", (3, 8, 8, 8, 4), 4, 2, 0, 12, 6, 2,
                dict(beta=0.5, tau=-1.0, lr=0.05, lambda_lr=0.04, kappa_lr=1e-3, max_corrections=1), seed=12,
                kappa_init=5)
    trainer_run("ref_k1_alm", (2, 6, 6, 6, 3), 1, 2, 0, 10, 10, 4,
                dict(beta=1.0, tau=-1.0, lr=0.05, lambda_lr=0.05, kappa_lr=1e-9, max_corrections=1), seed=13)
    trainer_run("ref_k3_l1_tau", (3, 5, 5, 6, 3), 3, 1, 1, 8, 8, 2,
                dict(beta=2.0, tau=1e-6, lr=0.05, lambda_lr=0.02, kappa_lr=1e-9, max_corrections=3), seed=14)
    trainer_run("ref_k2_linf", (3, 5, 5, 4, 3), 2, 1, 2, 8, 8, 2,
                dict(beta=2.0, tau=-1.0, lr=0.05, lambda_lr=0.02, kappa_lr=1e-9, max_corrections=1), seed=15)
    pieces("ref_pieces")
    # d = h = 64: at H = W = 1 these hit the device's tcgen05 plane path (C = hidden = 64), so
    # reference-held vectors pin the plane kernels, including stage 0 under a perturbed lambda
    trainer_run("ref_k4_alm_d64", (3, 64, 64, 8, 10), 4, 2, 0, 32, 16, 2,
                dict(beta=0.5, tau=-1.0, lr=0.05, lambda_lr=0.05, kappa_lr=1e-4, max_corrections=1), seed=21,
                kappa_init=22, lam_perturb=0.1)
    trainer_run("ref_k2_penalty_d64", (3, 64, 64, 4, 10), 2, 1, 0, 24, 24, 3,
                dict(beta=1.0, tau=-1.0, lr=0.05, lambda_lr=0.05, kappa_lr=1e-9, max_corrections=1), seed=23,
                lam_perturb=0.2)
    pieces("ref_pieces_d64", seed=24, dims=(3, 64, 64, 6, 10), K=3, N=16)
    serial("ref_serial")
    psi_kats("ref_psi")
