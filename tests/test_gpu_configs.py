"""GPU parity at the BASELINE configurations, against the oracle restated
over torch fp64 (oracle/respar_torch64.py, pinned to the numpy oracle and through it to the
compiled reference): the bench's own networks, batch, stages, mode and step parameters
(bench.py step_params), on the reference's synthetic data stream.

* C2 at full size (B 256, 3x32x32, C 64, L 16, K 4, ALM): one iteration compared quantity by
  quantity, and the loss curve of 20 iterations tracking the oracle's;
* C3 (L 64, K 8) at B 32, and its loss curve over 10 iterations at B 16; C4 (serial, the same
  64-block network) at B 16;
* C1 (1x28x28, C 16: the SIMT conv path) at full size;
* C5 (C 256, bf16 operands with fp32 accumulation) at full width, B 4.

Tolerances: fp32 math -- loss, lambda, X_end 1e-4 (FP32_TOL) max-norm relative per tensor,
the gradient-derived quantities (gradients, kappa, p) DERIVED_TOL (tests/test_gpu_plane_parity.py);
bf16 math -- 2e-2 (BF16_TOL), loss 1e-3.
"""
import ctypes as C

import numpy as np
import pytest

import bench
import paper_2009_01462_b200 as rp
from oracle import respar_oracle as O
from tests.helpers import FP32_TOL, rel_err, split_params

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
T = pytest.importorskip("oracle.respar_torch64")
from paper_2009_01462_b200._lib import lib  # noqa: E402

# the fp32 floor run must be plain fp32 (torch would otherwise run fp32 convs / matmuls as TF32)
torch.backends.cudnn.allow_tf32 = False
torch.backends.cuda.matmul.allow_tf32 = False

DERIVED_TOL = 1e-3
BF16_TOL = 2e-2


def _setup(name, B=None, L=None):
    cfg = dict(bench.CONFIGS[name])
    if B:
        cfg["B"] = B
    if L:
        cfg["L"] = L
    og = O.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], bench.CLASSES)
    net = O.make_net(og, O.Rng(bench._splitmix(1)))
    p32 = net.flat().astype(np.float32)
    x, y = O.synthetic_batch(og, cfg["B"], seed=1000)
    x32 = np.ascontiguousarray(x, np.float32)
    sp = bench.step_params(cfg)
    osp = O.StepParams(beta=sp.beta, tau=sp.tau, lr=sp.lr, lambda_lr=sp.lambda_lr, kappa_lr=sp.kappa_lr,
                       max_corrections=sp.max_corrections)
    g = rp.Geometry(og.in_channels, og.height, og.width, og.channels, og.hidden, og.blocks, og.classes)
    return cfg, og, p32, x32, y, sp, osp, g


def _oracle(og, p32, x32, cfg, K, dtype=None):
    dev = torch.device("cuda")
    dtype = dtype or torch.float64
    mode = T.ALM if cfg["mode"] == "alm" else T.PENALTY
    tr = T.DecoupledTrainer(T.Net(og, p32.astype(np.float64), dev, dtype), K, mode, T.SQUARED_L2, cfg["B"])
    xt = torch.from_numpy(x32.astype(np.float64)).to(device=dev, dtype=dtype)
    tr.reset_lambda_from_forward(xt)
    return tr, xt


def _close_derived(got, want, want32, tol=DERIVED_TOL, factor=16.0):
    """max(tol |want|, factor x the error of a plain fp32 execution): kappa, p and the early
    stages' gradients are formed from lambda - X_end, whose difference after a stationary start
    (reset_lambda_from_forward) sits at the fp32 rounding level of X_end itself -- in any fp32
    implementation; the plane path's X_end carries ~8x fp32's rounding (tcgen05 accumulation),
    hence the factor."""
    got = np.asarray(got, np.float64).reshape(-1)
    want = np.asarray(want, np.float64).reshape(-1)
    w32 = np.asarray(want32, np.float64).reshape(-1)
    err = float(np.abs(got - want).max()) if want.size else 0.0
    bound = max(tol * float(np.abs(want).max()), factor * float(np.abs(w32 - want).max())) if want.size else 0.0
    return err <= bound or err == 0.0, (err, bound)


def test_c2_full_size_one_iteration_and_20_step_loss_curve():
    cfg, og, p32, x32, y, sp, osp, g = _setup("C2")
    K, B = cfg["K"], cfg["B"]
    gt = rp.DecoupledTrainer(g, K, rp.ALM, rp.SQUARED_L2, B, params=p32)
    gt.reset_lambda_from_forward(x32)
    ot, xt = _oracle(og, p32, x32, cfg, K)
    o32, xt32 = _oracle(og, p32, x32, cfg, K, torch.float32)
    yt = torch.from_numpy(y.astype(np.int64)).cuda()
    xd = torch.from_numpy(x32).cuda()
    yd = torch.from_numpy(y.astype(np.int32)).cuda()
    # iteration 1, quantity by quantity
    lg = gt.step_device(xd.data_ptr(), yd.data_ptr(), B, 0, sp, read_loss=True)
    lo = ot.step(xt, yt, 0, osp)
    o32.step(xt32, yt, 0, osp)
    assert abs(lg - lo) <= FP32_TOL * abs(lo), (lg, lo)
    ranges = O.partition(og.blocks, K)
    want_g = T.grads_flat(og, ot.last_grads, ranges)
    want_g32 = T.grads_flat(og, o32.last_grads, ranges)
    got_g = gt.grads().astype(np.float64)
    for (nm, a), (_, b), (_, c) in zip(split_params(og, got_g), split_params(og, want_g), split_params(og, want_g32)):
        ok, e = _close_derived(a, b, c)
        assert ok, ("grad", nm, e)
    # the last stage's update (the only one a stationary start moves in iteration 1)
    beg = int(lib().rp_param_offset_block(C.byref(g.c()), og.blocks - og.blocks // K))
    d_got = gt.params()[beg:].astype(np.float64) - p32[beg:]
    d_want = ot.net.flat()[beg:] - p32[beg:].astype(np.float64)
    assert rel_err(d_got, d_want) <= DERIVED_TOL, rel_err(d_got, d_want)
    for k in range(K):
        assert rel_err(gt.state(k, rp.BOUNDARY_OUT), ot.bout[k].cpu().numpy()) <= FP32_TOL, k
        ok, e = _close_derived(gt.state(k, rp.BOUNDARY_ADJOINT), ot.badj[k].cpu().numpy(), o32.badj[k].cpu().numpy())
        assert ok, ("p", k, e)
        if k > 0:
            assert rel_err(gt.state(k, rp.LAMBDA), ot.lam[k].cpu().numpy()) <= FP32_TOL, k
            ok, e = _close_derived(gt.state(k, rp.KAPPA), ot.kappa[k].cpu().numpy(), o32.kappa[k].cpu().numpy())
            assert ok, ("kappa", k, e)
    # iterations 2..20: the loss curves track each other
    lgs, los = [lg], [lo]
    for _ in range(19):
        lgs.append(gt.step_device(xd.data_ptr(), yd.data_ptr(), B, 0, sp, read_loss=True))
        los.append(ot.step(xt, yt, 0, osp))
    errs = [abs(a - b) / abs(b) for a, b in zip(lgs, los)]
    print("C2 loss curve (gpu, oracle, rel):", [(round(a, 6), round(b, 6), f"{e:.1e}") for a, b, e in
                                                zip(lgs, los, errs)])
    assert max(errs) <= FP32_TOL, max(errs)
    assert los[-1] < los[0]   # the synthetic batch is being fitted
    assert rel_err(gt.params(), ot.net.flat()) <= FP32_TOL


@pytest.mark.parametrize("name,B", [("C3", 32), ("C1", None)])
def test_config_three_iterations(name, B):
    cfg, og, p32, x32, y, sp, osp, g = _setup(name, B=B)
    K, B = cfg["K"], cfg["B"]
    mode = rp.ALM if cfg["mode"] == "alm" else rp.PENALTY
    gt = rp.DecoupledTrainer(g, K, mode, rp.SQUARED_L2, B, params=p32)
    gt.reset_lambda_from_forward(x32)
    ot, xt = _oracle(og, p32, x32, cfg, K)
    o32, xt32 = _oracle(og, p32, x32, cfg, K, torch.float32)
    yt = torch.from_numpy(y.astype(np.int64)).cuda()
    lg, lo = [], []
    for _ in range(3):
        lg.append(gt.step(x32, y, 0, sp))
        lo.append(ot.step(xt, yt, 0, osp))
        o32.step(xt32, yt, 0, osp)
    assert rel_err(lg, lo) <= FP32_TOL, (lg, lo)
    assert rel_err(gt.params(), ot.net.flat()) <= FP32_TOL
    for k in range(K):
        assert rel_err(gt.state(k, rp.BOUNDARY_OUT), ot.bout[k].cpu().numpy()) <= FP32_TOL, k
        if k > 0:
            assert rel_err(gt.state(k, rp.LAMBDA), ot.lam[k].cpu().numpy()) <= FP32_TOL, k
    ranges = O.partition(og.blocks, K)
    want_g = T.grads_flat(og, ot.last_grads, ranges)
    want_g32 = T.grads_flat(og, o32.last_grads, ranges)
    for (nm, a), (_, b), (_, c) in zip(split_params(og, gt.grads().astype(np.float64)), split_params(og, want_g),
                                       split_params(og, want_g32)):
        ok, e = _close_derived(a, b, c)
        assert ok, (name, "grad", nm, e)


def test_c3_ten_step_loss_curve():
    """C3's 64-block, 8-stage network (conv_pm CTA pairs on every fprop / dgrad, the paired plane
    wgrad) at B 16: the loss curve of 10 iterations tracks the fp64 oracle's at FP32_TOL, and
    the parameters after them too."""
    cfg, og, p32, x32, y, sp, osp, g = _setup("C3", B=16)
    K, B = cfg["K"], cfg["B"]
    gt = rp.DecoupledTrainer(g, K, rp.ALM, rp.SQUARED_L2, B, params=p32)
    gt.reset_lambda_from_forward(x32)
    ot, xt = _oracle(og, p32, x32, cfg, K)
    yt = torch.from_numpy(y.astype(np.int64)).cuda()
    lg, lo = [], []
    for _ in range(10):
        lg.append(gt.step(x32, y, 0, sp))
        lo.append(ot.step(xt, yt, 0, osp))
    errs = [abs(a - b) / abs(b) for a, b in zip(lg, lo)]
    print("C3 loss curve (gpu, oracle, rel):", [(round(a, 6), round(b, 6), f"{e:.1e}") for a, b, e in zip(lg, lo, errs)])
    assert max(errs) <= FP32_TOL, max(errs)
    assert rel_err(gt.params(), ot.net.flat()) <= FP32_TOL


def test_c4_serial_64_blocks():
    """C4: serial full backprop (serial_train_step, network.cpp:236-244) of the C3 network."""
    cfg, og, p32, x32, y, sp, osp, g = _setup("C4", B=16)
    B = cfg["B"]
    st = rp.SerialTrainer(g, B, params=p32)
    ot, xt = _oracle(og, p32, x32, cfg, 1)
    yt = torch.from_numpy(y.astype(np.int64)).cuda()
    lr = cfg["lr"]
    for _ in range(3):
        lg = st.serial_train_step(x32, y, lr)
        lo = ot.step(xt, yt, 0, O.StepParams(beta=1.0, lr=lr, lambda_lr=0.0, kappa_lr=0.0))
        assert abs(lg - lo) <= FP32_TOL * abs(lo), (lg, lo)
    assert rel_err(st.params(), ot.net.flat()) <= FP32_TOL


def test_c5_full_width_bf16():
    """C5: C = 256, 64 blocks, K = 8, bf16 operands / fp32 accumulation, at B = 4."""
    cfg, og, p32, x32, y, sp, osp, g = _setup("C5", B=4)
    K, B = cfg["K"], cfg["B"]
    gt = rp.DecoupledTrainer(g, K, rp.ALM, rp.SQUARED_L2, B, params=p32, math="bf16")
    gt.reset_lambda_from_forward(x32)
    ot, xt = _oracle(og, p32, x32, cfg, K)
    yt = torch.from_numpy(y.astype(np.int64)).cuda()
    lg, lo = [], []
    for _ in range(2):
        lg.append(gt.step(x32, y, 0, sp))
        lo.append(ot.step(xt, yt, 0, osp))
    assert rel_err(lg, lo) <= 1e-3, (lg, lo)
    for k in range(K):
        assert rel_err(gt.state(k, rp.BOUNDARY_OUT), ot.bout[k].cpu().numpy()) <= BF16_TOL, k
    # the last stage's update (a stationary start moves the others by amounts below fp32 resolution)
    beg = int(lib().rp_param_offset_block(C.byref(g.c()), og.blocks - og.blocks // K))
    d_got = gt.params()[beg:].astype(np.float64) - p32[beg:]
    d_want = ot.net.flat()[beg:] - p32[beg:].astype(np.float64)
    print("C5 last-stage update error:", rel_err(d_got, d_want))
    assert rel_err(d_got, d_want) <= BF16_TOL
