"""GPU parity of the fp32 plane path (tcgen05 convs fed by bf16 plane pairs, C = hidden = 64 --
the kernels every BASELINE fp32 config runs) against the reference and the fp64 oracle, in
states where every stage's synthetic loss is live: lambda perturbed off the forward states
and kappa non-zero, over several iterations, comparing per-stage gradients, parameter
*deltas*, lambda, kappa, the boundary adjoints p and the losses.

Tolerances (north_star: "1e-4 relative after one iteration, loss curves tracking over N
iterations"): FP32_TOL = 1e-4 max-norm relative per tensor for loss, lambda, X_end.
Gradients, parameter deltas, kappa and p are sums over many positions of products of
cotangents formed from differences of nearly equal boundary states; their bound is
max(DERIVED_TOL |want|, 8 x the error a plain fp32 execution of the same algorithm makes)
(``fp32_close``), the floor measured by running the oracle in fp32 beside it
(tools/plane_err_table.py prints both columns).

Also the reference's algorithm invariants on this path (test_decoupled.cpp): serial-adjoint
consistency (187-221), the stationarity identity (270-307), the monotone beta response
(329-351), stage locality (353-375) and the per-stage parameter slice (377-397).
"""
import ctypes as C

import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from oracle import respar_oracle as O
from paper_2009_01462_b200._lib import lib
from tests.helpers import FP32_TOL, dense_geometry, load, param_rel_errs, rel_err, split_params

pytestmark = pytest.mark.gpu

# bound for the gradient-derived quantities (grads, deltas, kappa, p): the plane operands carry
# 16 significant bits (bf16 pair), whose per-product error (~2^-17) reaches 1e-4..5e-4 max-norm
# relative on gradients after cancellation (tools/plane_err_table.py)
DERIVED_TOL = 1e-3


def geo(og: O.Geometry) -> rp.Geometry:
    return rp.Geometry(og.in_channels, og.height, og.width, og.channels, og.hidden, og.blocks, og.classes,
                       og.activation, og.step_h)


def on_plane_path(og, nrows):
    g = geo(og).c()
    return lib().rp_op_block_planes_supported(C.byref(g), nrows, rp.MATH["fp32"]) == 1


def fp32_close(got, want, want32, tol=DERIVED_TOL, factor=8.0):
    got = np.asarray(got, np.float64).reshape(-1)
    want = np.asarray(want, np.float64).reshape(-1)
    w32 = np.asarray(want32, np.float64).reshape(-1)
    if want.size == 0:
        return True, (0.0, 0.0)
    err = float(np.abs(got - want).max())
    bound = max(tol * float(np.abs(want).max()), factor * float(np.abs(w32 - want).max()))
    return err <= bound or err == 0.0, (err, bound)


def per_tensor_close(og, got, want, want32, what):
    """fp32_close on every parameter tensor of the flat layout (skipping all-zero ones)."""
    for (n, a), (_, b), (_, c) in zip(split_params(og, got), split_params(og, want), split_params(og, want32)):
        if np.abs(b).max() == 0.0 and np.abs(a).max() == 0.0:
            continue
        ok, info = fp32_close(a, b, c)
        assert ok, (what, n, info)


# --------------------------------------------- reference-generated goldens at d = 64
@pytest.mark.parametrize("name", ["ref_k4_alm_d64", "ref_k2_penalty_d64"])
def test_d64_trainer_vs_reference_golden(name):
    """The compiled reference's own trajectory (tests/golden/make_golden.py) with lambda
    perturbed and kappa non-zero, replayed on the tcgen05 plane path (d = h = 64 at
    H = W = 1 is the reference's dense net)."""
    f = load(name)
    og = dense_geometry(f["dims"])
    K, mode, kind, N = int(f["K"]), int(f["mode"]), int(f["penalty"]), int(f["N"])
    assert on_plane_path(og, int(f["batch"]))
    p0 = O.embed_dense_params(og, f["params0"]).astype(np.float32)
    tr = rp.DecoupledTrainer(geo(og), K, mode, kind, N, params=p0)
    x = f["x"].astype(np.float32).reshape(N, 1, 1, og.in_channels)
    tr.reset_lambda_from_forward(x)
    for k in range(1, K):
        tr.set_state(k, rp.LAMBDA, f[f"lam0_{k}"].reshape(N, 1, 1, og.channels))
        tr.set_state(k, rp.KAPPA, f[f"kappa0_{k}"].reshape(N, 1, 1, og.channels))
    beta, tau, lr, llr, klr, mc = f["sp"]
    sp = rp.StepParams(beta, tau, lr, llr, klr, int(mc))
    losses = []
    b = int(f["batch"])
    for _ in range(int(f["epochs"])):
        for r0 in range(0, N, b):
            nr = min(b, N - r0)
            losses.append(tr.step(x[r0:r0 + nr], f["y"][r0:r0 + nr], r0, sp))
    assert rel_err(losses, f["losses"]) <= FP32_TOL, (losses, f["losses"])
    got = O.extract_dense_params(og, tr.params().astype(np.float64))
    want, start = f["params"], f["params0"]
    # the update itself (not the parameters it is added to): max-norm relative per run
    assert rel_err(got - start, want - start) <= 5 * FP32_TOL, rel_err(got - start, want - start)
    assert rel_err(got, want) <= FP32_TOL
    for k in range(K):
        for nm, which in (("lam", rp.LAMBDA), ("kappa", rp.KAPPA), ("bout", rp.BOUNDARY_OUT),
                          ("badj", rp.BOUNDARY_ADJOINT)):
            key = f"{nm}_{k}"
            if key in f:
                err = rel_err(tr.state(k, which).reshape(N, -1), f[key])
                assert err <= (5 * FP32_TOL if nm in ("kappa", "badj") else FP32_TOL), (key, err)


def test_d64_pieces_vs_reference_golden():
    """stage_backward_update gradients of every stage (stage 0 included) under a frozen
    snapshot with perturbed lambda and non-zero kappa, from the reference (decoupled.cpp:85-115),
    on the plane path: the synthetic upstream and its bf16 plane pair feed the first conv."""
    f = load("ref_pieces_d64")
    og = dense_geometry(f["dims"])
    K, N = int(f["K"]), int(f["N"])
    assert on_plane_path(og, N)
    tr = rp.DecoupledTrainer(geo(og), K, rp.ALM, rp.SQUARED_L2, N,
                             params=O.embed_dense_params(og, f["params0"]).astype(np.float32))
    x = f["x"].astype(np.float32).reshape(N, 1, 1, -1)
    tr.reset_lambda_from_forward(x)
    for k in range(1, K):
        tr.set_state(k, rp.LAMBDA, f[f"lam_in_{k}"].reshape(N, 1, 1, -1))
        tr.set_state(k, rp.KAPPA, f[f"kappa_in_{k}"].reshape(N, 1, 1, -1))
    beta, lr = float(f["beta"]), float(f["lr"])
    for k in range(K):
        if k + 1 < K:
            tr.take_snapshot(k, 0, N)
        tr.stage_forward(k, x if k == 0 else None, 0, nrows=N)
        assert rel_err(tr.state(k, rp.BOUNDARY_OUT).reshape(N, -1), f[f"bout_{k}"]) <= FP32_TOL
        g = tr.stage_backward_update(k, f["y"] if k == K - 1 else None, beta, lr, 0)
        want = f[f"grads_{k}"]
        got = O.extract_dense_params(og, g.astype(np.float64))
        mask = want != 0
        assert mask.sum() > 0
        assert rel_err(got[mask], want[mask]) <= FP32_TOL, (k, rel_err(got[mask], want[mask]))
        assert rel_err(tr.state(k, rp.BOUNDARY_ADJOINT).reshape(N, -1), f[f"badj_{k}"]) <= FP32_TOL
    for k in range(1, K):
        assert rel_err(tr.correction_gradient(k, beta, 0, N).reshape(N, -1), f[f"corrgrad_{k}"]) <= FP32_TOL
        tr.correct_aux(k, rp.StepParams(beta=beta, tau=-1.0, lambda_lr=0.3), 0, N)
        assert rel_err(tr.state(k, rp.LAMBDA).reshape(N, -1), f[f"lam_corr_{k}"]) <= FP32_TOL
        tr.correct_multiplier(k, beta, 1e-3, 0, N)
        assert rel_err(tr.state(k, rp.KAPPA).reshape(N, -1), f[f"kappa_corr_{k}"]) <= FP32_TOL


# ------------------------------------------------ 3x3 plane path vs the fp64 oracle
PLANE_CASES = [
    # (geometry, K, mode, N, batch, steps)
    (O.Geometry(3, 8, 8, 64, 64, 8, 10), 2, O.ALM, 8, 8, 3),
    (O.Geometry(3, 8, 8, 64, 64, 8, 10), 4, O.ALM, 8, 4, 3),                 # mini-batches (row0 > 0)
    (O.Geometry(3, 8, 8, 64, 64, 8, 10), 4, O.PENALTY, 6, 6, 3),
    (O.Geometry(3, 6, 10, 64, 64, 4, 10, step_h=0.5), 2, O.ALM, 5, 5, 3),    # ragged frame, h != 1
    (O.Geometry(3, 8, 8, 64, 64, 4, 10, activation=O.IDENTITY), 2, O.ALM, 4, 4, 3),
    (O.Geometry(3, 32, 32, 64, 64, 4, 10), 4, O.ALM, 4, 4, 3),               # C2's image and channels
]


def perturbed_run(og, K, mode, N, batch, steps, seed=3, lam_scale=0.1):
    """fp64 oracle (truth), fp32 oracle (the noise floor) and the device, from the same
    fp32-rounded parameters and inputs, with lambda_k += U(-s, s) and kappa_k ~ the size of
    the penalty term, so every stage's upstream mixes both parts of decoupled.cpp:105-110."""
    net = O.make_net(og, O.Rng(seed))
    for l in range(og.blocks):
        net.b1[l][...] = O.rng_uniform(O.Rng(100 + l), og.hidden, -0.1, 0.1)
        net.b2[l][...] = O.rng_uniform(O.Rng(200 + l), og.channels, -0.1, 0.1)
    net.s_b[...] = O.rng_uniform(O.Rng(300), og.channels, -0.1, 0.1)
    net.t_b[...] = O.rng_uniform(O.Rng(301), og.classes, -0.1, 0.1)
    p32 = net.flat().astype(np.float32)
    net.load_flat(p32.astype(np.float64))
    x, y = O.synthetic_batch(og, N, seed=seed + 7)
    x32 = x.astype(np.float32)
    x = x32.astype(np.float64)
    beta = 0.5
    ot = O.DecoupledTrainer(net, K, mode, O.SQUARED_L2, N)
    o32 = O.DecoupledTrainer(net.astype(np.float32), K, mode, O.SQUARED_L2, N)
    gt = rp.DecoupledTrainer(geo(og), K, mode, rp.SQUARED_L2, N, params=p32)
    ot.reset_lambda_from_forward(x)
    o32.reset_lambda_from_forward(x32)
    gt.reset_lambda_from_forward(x32)
    kscale = beta / (batch * og.feature_size) * 2 * lam_scale
    prng = O.Rng(seed + 50)
    for k in range(1, K):
        lam = (ot.stage(k).lam + O.rng_uniform(prng, ot.stage(k).lam.size, -lam_scale, lam_scale)
               .reshape(ot.stage(k).lam.shape)).astype(np.float32)
        kap = (O.rng_uniform(prng, lam.size, -kscale, kscale).reshape(lam.shape)).astype(np.float32)
        for t, dt in ((ot, np.float64), (o32, np.float32)):
            t.stage(k).lam[...] = lam.astype(dt)
            t.stage(k).kappa[...] = kap.astype(dt)
        gt.set_state(k, rp.LAMBDA, lam)
        gt.set_state(k, rp.KAPPA, kap)
    sp_o = O.StepParams(beta=beta, lr=0.05, lambda_lr=0.05, kappa_lr=1e-3 * 2 * beta / (batch * og.feature_size))
    sp_g = rp.StepParams(beta=beta, lr=0.05, lambda_lr=0.05, kappa_lr=sp_o.kappa_lr)
    lo, lg = [], []
    for _ in range(steps):
        for r0 in range(0, N, batch):
            nr = min(batch, N - r0)
            lo.append(ot.step(x[r0:r0 + nr], y[r0:r0 + nr], r0, sp_o))
            o32.step(x32[r0:r0 + nr], y[r0:r0 + nr], r0, sp_o)
            lg.append(gt.step(x32[r0:r0 + nr], y[r0:r0 + nr], r0, sp_g))
    return dict(ot=ot, o32=o32, gt=gt, lo=np.array(lo), lg=np.array(lg), p0=p32.astype(np.float64))


@pytest.mark.parametrize("case", range(len(PLANE_CASES)))
def test_plane_trainer_perturbed_vs_oracle(case):
    og, K, mode, N, batch, steps = PLANE_CASES[case]
    assert on_plane_path(og, batch)
    r = perturbed_run(og, K, mode, N, batch, steps)
    ot, o32, gt = r["ot"], r["o32"], r["gt"]
    assert rel_err(r["lg"], r["lo"]) <= FP32_TOL, (r["lg"], r["lo"])
    ranges = O.partition(og.blocks, K)
    # per-stage gradients of the last iteration (rp_trainer_get_grads vs the oracle's NetGrads);
    # stage 0's are non-zero because its synthetic loss is live
    want_g = O.grads_flat(og, ot.last_grads, ranges)
    want_g32 = O.grads_flat(og, o32.last_grads, ranges)
    got_g = gt.grads().astype(np.float64)
    s0 = [a for (n, a) in split_params(og, want_g) if n.startswith("b0.") or n.startswith("s.")]
    assert max(np.abs(a).max() for a in s0) > 0.0
    per_tensor_close(og, got_g, want_g, want_g32, "grads")
    # the parameter updates accumulated over the run, per tensor
    got_p, want_p, want_p32 = gt.params().astype(np.float64), ot.net.flat(), o32.net.flat().astype(np.float64)
    per_tensor_close(og, got_p - r["p0"], want_p - r["p0"], want_p32 - r["p0"], "deltas")
    errs = param_rel_errs(og, got_p, want_p)
    assert max(errs.values()) <= FP32_TOL, errs
    for k in range(K):
        st, s32 = ot.stage(k), o32.stage(k)
        for which, want, w32 in ((rp.LAMBDA, st.lam, s32.lam), (rp.KAPPA, st.kappa, s32.kappa),
                                 (rp.BOUNDARY_OUT, st.boundary_out, s32.boundary_out),
                                 (rp.BOUNDARY_ADJOINT, st.boundary_adjoint, s32.boundary_adjoint)):
            if k == 0 and which in (rp.LAMBDA, rp.KAPPA):
                continue
            got = gt.state(k, which)
            if which in (rp.LAMBDA, rp.BOUNDARY_OUT):
                assert rel_err(got, want) <= FP32_TOL, (k, which, rel_err(got, want))
            else:
                ok, info = fp32_close(got, want, w32)
                assert ok, (k, which, info)


# ------------------------------------------------------ algorithm invariants on device
INV_GEO = O.Geometry(3, 8, 8, 64, 64, 8, 10)


def stage_param_range(og, K, k):
    """Stage k's slice of the flat parameters: its blocks, plus S (k = 0) and T (k = K-1)
    (network.cpp:174-191, the device trainer's Layout)."""
    g = geo(og).c()
    n = og.blocks // K
    beg = 0 if k == 0 else int(lib().rp_param_offset_block(C.byref(g), k * n))
    end = O.param_count(og) if k == K - 1 else int(lib().rp_param_offset_block(C.byref(g), (k + 1) * n))
    return beg, end


def _inv_net(seed):
    net = O.make_net(INV_GEO, O.Rng(seed))
    p32 = net.flat().astype(np.float32)
    net.load_flat(p32.astype(np.float64))
    return net, p32


@pytest.mark.parametrize("K", [2, 4])
def test_serial_adjoint_consistency_on_planes(K):
    """test_decoupled.cpp:187-221: lambda_k = serial X_{kn}, kappa_k = serial adjoint at kn;
    every stage's frozen-snapshot gradients then equal serial backprop's -- both the device
    serial trainer's and the fp64 oracle's."""
    og, N = INV_GEO, 6
    net, p32 = _inv_net(7)
    x, y = O.synthetic_batch(og, N, seed=8)
    x32 = x.astype(np.float32)
    x = x32.astype(np.float64)
    n = og.blocks // K
    # fp64 serial trace: the adjoint at every block boundary
    tape = O.net_forward(net, x, 0, og.blocks)
    _, up = O.loss_phi(tape.logits, y)
    cot, full = O.net_vjp(net, tape, up)
    adj = {og.blocks: None}
    g_t = up @ net.t_w.T
    c = np.broadcast_to(g_t[:, None, None, :] / (og.height * og.width), tape.features.shape).copy()
    adj[og.blocks] = c
    for l in range(og.blocks - 1, -1, -1):
        c, _ = O.block_vjp(net, l, tape.blocks[l], c)
        adj[l] = c
    want = O.grads_flat(og, [full], [(0, og.blocks)])
    # device serial gradients
    ser = rp.SerialTrainer(geo(og), N, params=p32)
    ser.serial_train_step(x32, y, 0.0)
    dev_serial = ser.grads().astype(np.float64)
    assert rel_err(dev_serial, want) <= FP32_TOL
    tr = rp.DecoupledTrainer(geo(og), K, rp.ALM, rp.SQUARED_L2, N, params=p32)
    tr.reset_lambda_from_forward(x32)                                  # lambda_k := X_{kn}
    for k in range(1, K):
        tr.set_state(k, rp.KAPPA, adj[k * n].astype(np.float32))
    got = np.zeros_like(want)
    for k in range(K):
        if k + 1 < K:
            tr.take_snapshot(k, 0, N)
        tr.stage_forward(k, x32 if k == 0 else None, 0, nrows=N)
        g = tr.stage_backward_update(k, y if k == K - 1 else None, 3.7, 0.0, 0).astype(np.float64)
        beg, end = stage_param_range(og, K, k)
        got[beg:end] = g[beg:end]
        assert rel_err(tr.state(k, rp.BOUNDARY_ADJOINT), adj[k * n]) <= FP32_TOL, k
    for (nm, a), (_, b_), (_, c_) in zip(split_params(og, got), split_params(og, want), split_params(og, dev_serial)):
        assert rel_err(a, b_) <= FP32_TOL, (K, nm, rel_err(a, b_))
        assert rel_err(a, c_) <= FP32_TOL, (K, nm, rel_err(a, c_))


def test_stationarity_identity_on_planes():
    """test_decoupled.cpp:270-307: frozen net (lr 0), frozen multiplier (kappa_lr 0); at the
    correction fixed point lambda - X == (#/2 beta)(kappa - p).  beta and lambda_lr are scaled
    to the conv normaliser # = N H W C so the fixed-point iteration contracts as in the
    reference's dense test."""
    og, N, K = O.Geometry(3, 8, 8, 64, 64, 4, 10), 4, 2
    p32 = O.make_net(og, O.Rng(10)).flat().astype(np.float32)
    x, y = O.synthetic_batch(og, N, seed=10)
    x32 = x.astype(np.float32)
    norm = N * og.feature_size
    beta = norm / 2.0 / 8.0                       # #/(2 beta) = 8
    for with_kappa in (False, True):
        tr = rp.DecoupledTrainer(geo(og), K, rp.ALM if with_kappa else rp.PENALTY, rp.SQUARED_L2, N, params=p32)
        tr.reset_lambda_from_forward(x32)
        if with_kappa:
            tr.set_state(1, rp.KAPPA, O.rng_uniform(O.Rng(11), N * og.feature_size, -0.01, 0.01).astype(np.float32))
        sp = rp.StepParams(beta=beta, lr=0.0, lambda_lr=0.05 * 8.0, kappa_lr=0.0)   # contraction 0.95 / step
        for _ in range(800):
            tr.step(x32, y, 0, sp)
        tr.take_snapshot(0, 0, N)
        tr.stage_forward(0, x32, 0)
        tr.stage_backward_update(0, None, beta, 0.0, 0)
        tr.stage_forward(1, None, 0, nrows=N)
        tr.stage_backward_update(1, y, beta, 0.0, 0)
        lam = tr.state(1, rp.LAMBDA).astype(np.float64)
        xe = tr.state(0, rp.BOUNDARY_OUT).astype(np.float64)
        kap = tr.state(1, rp.KAPPA).astype(np.float64)
        p = tr.state(1, rp.BOUNDARY_ADJOINT).astype(np.float64)
        lhs = lam - xe
        rhs = (norm / (2.0 * beta)) * (kap - p)
        assert np.abs(lhs).max() > 0.0
        assert np.abs(lhs - rhs).max() <= 1e-3 * np.abs(lhs).max(), (with_kappa, np.abs(lhs - rhs).max(),
                                                                      np.abs(lhs).max())


def test_monotone_beta_response_on_planes():
    """test_decoupled.cpp:329-351: on the frozen subproblem a larger beta gives a smaller
    constraint violation."""
    og, N, K = O.Geometry(3, 8, 8, 64, 64, 4, 10), 4, 2
    p32 = O.make_net(og, O.Rng(12)).flat().astype(np.float32)
    x, y = O.synthetic_batch(og, N, seed=12)
    x32 = x.astype(np.float32)
    norm = N * og.feature_size
    prev = None
    for beta_ref in (1.0, 10.0, 100.0):
        beta = beta_ref * norm / 20.0             # the reference's # = 20: same contraction per step
        tr = rp.DecoupledTrainer(geo(og), K, rp.PENALTY, rp.SQUARED_L2, N, params=p32)
        tr.reset_lambda_from_forward(x32)
        sp = rp.StepParams(beta=beta, lr=0.0, lambda_lr=0.1)   # 2 lambda_lr beta / # = 0.01 beta_ref
        for _ in range(1500):
            tr.step(x32, y, 0, sp)
        tr.stage_forward(0, x32, 0)
        d = np.sqrt(((tr.state(1, rp.LAMBDA).astype(np.float64) -
                      tr.state(0, rp.BOUNDARY_OUT).astype(np.float64)) ** 2).sum())
        if prev is not None:
            assert d < prev, (beta_ref, d, prev)
        prev = d


def test_stage_locality_and_own_slice_on_planes():
    """test_decoupled.cpp:353-397: stage 0's backward reads only its tape and the snapshot
    (corrupting stage 1's master lambda / kappa afterwards changes nothing, bitwise), and its
    update touches only its own parameter slice."""
    og, N, K = INV_GEO, 5, 2
    _, p32 = _inv_net(13)
    x, y = O.synthetic_batch(og, N, seed=13)
    x32 = x.astype(np.float32)
    tr = rp.DecoupledTrainer(geo(og), K, rp.ALM, rp.SQUARED_L2, N, params=p32)
    tr.reset_lambda_from_forward(x32)
    tr.set_state(1, rp.LAMBDA, tr.state(1, rp.LAMBDA) + 0.3)
    tr.set_state(1, rp.KAPPA, O.rng_uniform(O.Rng(14), N * og.feature_size, -1e-4, 1e-4).astype(np.float32))
    tr.take_snapshot(0, 0, N)
    tr.stage_forward(0, x32, 0)
    first = tr.stage_backward_update(0, None, 2.0, 0.0, 0).copy()
    tr.set_state(1, rp.LAMBDA, np.full(N * og.feature_size, 1e9, np.float32))
    tr.set_state(1, rp.KAPPA, np.full(N * og.feature_size, -1e9, np.float32))
    tr.stage_forward(0, x32, 0)
    second = tr.stage_backward_update(0, None, 2.0, 0.1, 0)
    np.testing.assert_array_equal(first, second)
    after = tr.params()
    off = int(lib().rp_param_offset_block(C.byref(geo(og).c()), og.blocks // K))
    assert np.array_equal(after[off:], p32[off:])           # stage 1's blocks and the head untouched
    assert not np.array_equal(after[:off], p32[:off])       # stem and stage-0 blocks moved
