"""CPU: pin the oracle restatement (oracle/respar_oracle.py) to the reference.

1. against the committed golden vectors made by the reference itself
   (tests/golden/make_golden.py), <= 1e-12;
2. against the live reference library (oracle/_ref, built from /root/reference) on
   fresh random instances, when it is present;
3. the conv-specific parts (3x3 taps, GAP head) by central finite differences, the
   pattern of the reference's gradcheck.cpp:100-180 (eps 1e-5, rel-err floor 1e-3).
"""
import numpy as np
import pytest

from oracle import respar_oracle as O
from tests.helpers import dense_geometry, load, rel_err

TIGHT = 1e-12

TRAINER_FIXTURES = ["ref_k2_penalty", "ref_k4_alm_minibatch", "ref_k1_alm", "ref_k3_l1_tau", "ref_k2_linf",
                    "ref_k4_alm_d64", "ref_k2_penalty_d64"]


def run_oracle_fixture(f):
    g = dense_geometry(f["dims"])
    K, mode, kind, N = int(f["K"]), int(f["mode"]), int(f["penalty"]), int(f["N"])
    net = O.zero_net(g)
    net.load_flat(O.embed_dense_params(g, f["params0"]))
    tr = O.DecoupledTrainer(net, K, mode, kind, N)
    x = f["x"].reshape(N, 1, 1, g.in_channels)
    tr.reset_lambda_from_forward(x)
    for k in range(1, K):
        tr.stage(k).kappa[...] = f[f"kappa0_{k}"].reshape(N, 1, 1, g.channels)
        if f"lam0_{k}" in f:
            tr.stage(k).lam[...] = f[f"lam0_{k}"].reshape(N, 1, 1, g.channels)
    beta, tau, lr, llr, klr, mc = f["sp"]
    sp = O.StepParams(beta, tau, lr, llr, klr, int(mc))
    losses = []
    b = int(f["batch"])
    for _ in range(int(f["epochs"])):
        for r0 in range(0, N, b):
            nr = min(b, N - r0)
            losses.append(tr.step(x[r0:r0 + nr], f["y"][r0:r0 + nr], r0, sp))
    return g, tr, np.array(losses)


@pytest.mark.parametrize("name", TRAINER_FIXTURES)
def test_oracle_matches_reference_golden(name):
    f = load(name)
    g, tr, losses = run_oracle_fixture(f)
    assert rel_err(losses, f["losses"]) <= TIGHT
    assert rel_err(O.extract_dense_params(g, tr.net.flat()), f["params"]) <= TIGHT
    K = int(f["K"])
    for k in range(K):
        st = tr.stage(k)
        for nm, v in (("lam", st.lam), ("kappa", st.kappa), ("bout", st.boundary_out), ("badj", st.boundary_adjoint)):
            key = f"{nm}_{k}"
            if key in f:
                assert rel_err(v.reshape(f[key].shape), f[key]) <= 1e-11, key
    per, mx, _ = tr.violation_report()
    assert rel_err(per, f["violation"]) <= 1e-10


@pytest.mark.parametrize("name", ["ref_pieces", "ref_pieces_d64"])
def test_oracle_pieces_golden(name):
    f = load(name)
    g = dense_geometry(f["dims"])
    K, N = int(f["K"]), int(f["N"])
    net = O.zero_net(g)
    net.load_flat(O.embed_dense_params(g, f["params0"]))
    tr = O.DecoupledTrainer(net, K, O.ALM, O.SQUARED_L2, N)
    x = f["x"].reshape(N, 1, 1, -1)
    tr.reset_lambda_from_forward(x)
    for k in range(1, K):
        tr.stage(k).lam[...] = f[f"lam_in_{k}"].reshape(N, 1, 1, -1)
        tr.stage(k).kappa[...] = f[f"kappa_in_{k}"].reshape(N, 1, 1, -1)
    beta, lr = float(f["beta"]), float(f["lr"])
    for k in range(K):
        snap = tr.take_snapshot(k, 0, N) if k + 1 < K else None
        before = tr.net.flat()
        tr.stage_forward(k, x, 0)
        assert rel_err(tr.stage(k).boundary_out.reshape(N, -1), f[f"bout_{k}"]) <= TIGHT
        tr.stage_backward_update(k, f["y"], snap, beta, lr, 0)
        # NetGrads are recovered from the update: g = (before - after) / lr on the stage slice
        dense_g = O.extract_dense_params(g, (before - tr.net.flat()) / lr)
        mask = f[f"grads_{k}"] != 0
        assert rel_err(dense_g[mask], f[f"grads_{k}"][mask]) <= 1e-9
        assert rel_err(tr.stage(k).boundary_adjoint.reshape(N, -1), f[f"badj_{k}"]) <= TIGHT
    assert rel_err(O.extract_dense_params(g, tr.net.flat()), f["params1"]) <= TIGHT
    for k in range(1, K):
        assert rel_err(tr.correction_gradient(k, beta, 0, N).reshape(N, -1), f[f"corrgrad_{k}"]) <= TIGHT
        tr.correct_aux(k, O.StepParams(beta=beta, tau=-1.0, lambda_lr=0.3), 0, N)
        assert rel_err(tr.stage(k).lam.reshape(N, -1), f[f"lam_corr_{k}"]) <= TIGHT
        tr.correct_multiplier(k, beta, 1e-3, 0, N)
        assert rel_err(tr.stage(k).kappa.reshape(N, -1), f[f"kappa_corr_{k}"]) <= TIGHT


def test_oracle_serial_golden():
    f = load("ref_serial")
    g = dense_geometry(f["dims"])
    net = O.zero_net(g)
    net.load_flat(O.embed_dense_params(g, f["params0"]))
    x = f["x"].reshape(10, 1, 1, -1)
    losses = [O.serial_train_step(net, x, f["y"], float(f["lr"])) for _ in range(5)]
    assert rel_err(losses, f["losses"]) <= TIGHT
    assert rel_err(O.extract_dense_params(g, net.flat()), f["params"]) <= TIGHT


def test_oracle_psi_golden_and_kats():
    f = load("ref_psi")
    lam, x = np.array([[1.0, 2.0]]), np.zeros((1, 2))
    assert O.psi(O.SQUARED_L2, lam, x) == 5.0 == f["kat_psi_0"]       # test_penalty.cpp:32-38
    assert O.psi(O.L1, lam, x) == 3.0 == f["kat_psi_1"]
    assert O.psi(O.LINF, lam, x) == 2.0 == f["kat_psi_2"]
    assert np.array_equal(O.psi_grads(O.SQUARED_L2, lam, x)[0], [[2.0, 4.0]])
    for kind in range(3):
        assert O.psi(kind, f["a"], f["b"]) == pytest.approx(float(f[f"psi_{kind}"]), rel=1e-14)
        dl, dx = O.psi_grads(kind, f["a"], f["b"])
        assert np.array_equal(dl, f[f"dl_{kind}"])
        assert np.array_equal(dx, -dl)


def test_rng_closed_form():
    """draw i = mix(seed + (i+1) gamma) equals the sequential stream (tensor.cpp:163-185)."""
    r1, r2 = O.Rng(99), O.Rng(99)
    block = r1.next_u64_block(1000)
    seq = [r2.next_u64() for _ in range(1000)]
    assert [int(v) for v in block] == seq
    assert O.Rng(5).split().state == O.Rng(O.Rng(5).next_u64()).state


def _fd_check(f, x, analytic, eps=1e-5, floor=1e-3, n_probe=25, seed=0):
    """Central differences on a random subset of entries (gradcheck.cpp:16-32)."""
    rng = np.random.default_rng(seed)
    flat = x.reshape(-1)
    idx = rng.choice(flat.size, size=min(n_probe, flat.size), replace=False)
    worst = 0.0
    for i in idx:
        s = flat[i]
        flat[i] = s + eps
        hi = f()
        flat[i] = s - eps
        lo = f()
        flat[i] = s
        fd = (hi - lo) / (2 * eps)
        a = analytic.reshape(-1)[i]
        worst = max(worst, abs(a - fd) / max(abs(a), abs(fd), floor))
    return worst


def test_conv_oracle_gradcheck():
    """3x3-conv block VJP and GAP head vs FD (the conv analogue of gradcheck.cpp)."""
    g = O.Geometry(in_channels=2, height=4, width=5, channels=3, hidden=4, blocks=3, classes=3, step_h=0.7)
    net = O.make_net(g, O.Rng(3))
    for l in range(g.blocks):
        net.b1[l][...] = O.rng_uniform(O.Rng(10 + l), g.hidden, -0.2, 0.2)
        net.b2[l][...] = O.rng_uniform(O.Rng(20 + l), g.channels, -0.2, 0.2)
    x, y = O.synthetic_batch(g, 3, seed=4)

    def loss():
        return O.loss_phi(O.net_forward(net, x, 0, g.blocks).logits, y)[0]

    tape = O.net_forward(net, x, 0, g.blocks)
    _, gl = O.loss_phi(tape.logits, y)
    _, grads = O.net_vjp(net, tape, gl)
    worst = 0.0
    worst = max(worst, _fd_check(loss, net.s_w, grads.s_w))
    worst = max(worst, _fd_check(loss, net.t_w, grads.t_w))
    for l in range(g.blocks):
        gw1, gb1, gw2, gb2 = grads.blocks[l]
        worst = max(worst, _fd_check(loss, net.w1[l], gw1), _fd_check(loss, net.b1[l], gb1),
                    _fd_check(loss, net.w2[l], gw2), _fd_check(loss, net.b2[l], gb2))
    assert worst <= 1e-6

    # synthetic-loss input cotangent (stage k > 0): d/dlambda of (beta/#) psi + <kappa, X>
    lam = O.rng_uniform(O.Rng(7), 3 * g.feature_size, -1, 1).reshape(3, g.height, g.width, g.channels)
    lam_next = O.rng_uniform(O.Rng(8), lam.size, -1, 1).reshape(lam.shape)
    kap = O.rng_uniform(O.Rng(9), lam.size, -0.1, 0.1).reshape(lam.shape)
    beta, norm = 1.3, lam.size

    def syn():
        X = O.net_forward(net, lam, 1, 2).features
        return beta / norm * O.psi(O.SQUARED_L2, lam_next, X) + float((kap * X).sum())

    t2 = O.net_forward(net, lam, 1, 2)
    _, dx = O.psi_grads(O.SQUARED_L2, lam_next, t2.features)
    cot, _ = O.net_vjp(net, t2, beta / norm * dx + kap)
    assert _fd_check(syn, lam, cot) <= 1e-6


def test_oracle_degenerate_conv_equals_dense_kernel():
    """At H = W = 1 only the centre tap acts: non-centre weights have zero gradient."""
    g = O.Geometry(in_channels=3, height=1, width=1, channels=4, hidden=5, blocks=2, classes=3)
    net = O.make_net(g, O.Rng(1))
    x, y = O.synthetic_batch(g, 6, seed=2)
    tape = O.net_forward(net, x, 0, 2)
    _, gl = O.loss_phi(tape.logits, y)
    _, grads = O.net_vjp(net, tape, gl)
    for gw1, _, gw2, _ in grads.blocks:
        m = np.ones((3, 3), bool)
        m[1, 1] = False
        assert np.all(gw1[m] == 0) and np.all(gw2[m] == 0)


@pytest.mark.skipif(not __import__("oracle.refbind", fromlist=["x"]).available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("K,mode,kind", [(2, O.PENALTY, O.SQUARED_L2), (3, O.ALM, O.SQUARED_L2),
                                         (2, O.PENALTY, O.L1), (4, O.PENALTY, O.LINF)])
def test_oracle_vs_live_reference(K, mode, kind):
    from oracle import refbind as R
    dims = (2, 5, 4, 12, 3)
    rng = R.RefRng(100 + K)
    dense = R.make_net(rng, *dims)
    N = 10
    x = rng.uniform(N, 2, -1, 1)
    y = np.array([rng.next_u64() % 3 for _ in range(N)], np.int32)
    ref = R.RefTrainer(dims, 0, dense, K, mode, kind, N, workers=2)
    ref.reset_lambda_from_forward(x)
    g = dense_geometry(dims)
    net = O.zero_net(g)
    net.load_flat(O.embed_dense_params(g, dense))
    tr = O.DecoupledTrainer(net, K, mode, kind, N)
    xo = x.reshape(N, 1, 1, 2)
    tr.reset_lambda_from_forward(xo)
    sp = O.StepParams(beta=0.9, lr=0.05, lambda_lr=0.05, kappa_lr=1e-3)
    for _ in range(3):
        for r0 in (0, 5):
            a = ref.step(x[r0:r0 + 5], y[r0:r0 + 5], r0, beta=0.9, lr=0.05, lambda_lr=0.05, kappa_lr=1e-3)
            b = tr.step(xo[r0:r0 + 5], y[r0:r0 + 5], r0, sp)
            assert abs(a - b) <= 1e-12 * max(1.0, abs(a))
    assert rel_err(O.extract_dense_params(g, net.flat()), ref.params()) <= TIGHT


def test_torch64_oracle_matches_numpy_oracle():
    """oracle/respar_torch64.py (the BASELINE-size checker of tests/test_gpu_configs.py) is the
    numpy oracle restated over torch fp64: equal to it at 1e-12 over 3 ALM steps with lambda
    perturbed and kappa non-zero, for the step's loss, parameters, lambda, kappa, X_end and p."""
    import torch
    from oracle import respar_torch64 as T
    og = O.Geometry(3, 6, 5, 8, 8, 4, 10, step_h=0.7)
    net = O.make_net(og, O.Rng(3))
    x, y = O.synthetic_batch(og, 6, seed=4)
    K = 2
    on = O.DecoupledTrainer(net.copy(), K, O.ALM, O.SQUARED_L2, 6)
    tn = T.DecoupledTrainer(T.Net(og, net.flat(), "cpu"), K, T.ALM, T.SQUARED_L2, 6)
    on.reset_lambda_from_forward(x)
    tn.reset_lambda_from_forward(torch.from_numpy(x))
    rng = O.Rng(9)
    lam = on.stage(1).lam + O.rng_uniform(rng, on.stage(1).lam.size, -0.1, 0.1).reshape(on.stage(1).lam.shape)
    kap = O.rng_uniform(rng, lam.size, -1e-3, 1e-3).reshape(lam.shape)
    on.stage(1).lam[...] = lam
    on.stage(1).kappa[...] = kap
    tn.lam[1][...] = torch.from_numpy(lam)
    tn.kappa[1][...] = torch.from_numpy(kap)
    sp = O.StepParams(beta=0.5, lr=0.05, lambda_lr=0.05, kappa_lr=1e-3)
    yt = torch.from_numpy(y.astype(np.int64))
    for r0, nr in ((0, 6), (0, 3), (3, 3)):
        a = on.step(x[r0:r0 + nr], y[r0:r0 + nr], r0, sp)
        b = tn.step(torch.from_numpy(x[r0:r0 + nr]), yt[r0:r0 + nr], r0, sp)
        assert abs(a - b) <= 1e-12 * abs(a)
    assert rel_err(tn.net.flat(), on.net.flat()) <= 1e-12
    for k in range(K):
        assert rel_err(tn.bout[k].numpy(), on.stage(k).boundary_out) <= 1e-12
        assert rel_err(tn.badj[k].numpy(), on.stage(k).boundary_adjoint) <= 1e-11
    assert rel_err(tn.lam[1].numpy(), on.stage(1).lam) <= 1e-12
    assert rel_err(tn.kappa[1].numpy(), on.stage(1).kappa) <= 1e-11
    ranges = O.partition(og.blocks, K)
    assert rel_err(T.grads_flat(og, tn.last_grads, ranges), O.grads_flat(og, on.last_grads, ranges)) <= 1e-11
