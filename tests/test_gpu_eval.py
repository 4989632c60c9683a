"""GPU: evaluation on device (decoupled.cpp:332-347 -- the full serial forward, then loss_phi
and accuracy, network.cpp:193-234) against the fp64 oracle: the loss at 1e-4, the per-row
argmax (ties to the lowest class) bit-exact on every row whose oracle top-2 logit margin
exceeds the fp32 error bound, and the psi / psi_grads kernels against the reference's
golden vectors (penalty.cpp:38-87: L-inf first-index ties, sign(0) = 0)."""
import ctypes as C

import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from oracle import respar_oracle as O
from paper_2009_01462_b200._lib import lib
from tests.helpers import FP32_TOL, load

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _geo(og):
    return rp.Geometry(og.in_channels, og.height, og.width, og.channels, og.hidden, og.blocks, og.classes)


@pytest.mark.parametrize("og,N", [(O.Geometry(3, 8, 8, 64, 64, 4, 10), 200), (O.Geometry(3, 6, 6, 16, 16, 2, 10), 64),
                                  (O.Geometry(3, 1, 1, 64, 64, 4, 10), 300)])
def test_evaluate_on_device_matches_oracle(og, N):
    net = O.make_net(og, O.Rng(21))
    p32 = net.flat().astype(np.float32)
    net.load_flat(p32.astype(np.float64))
    x, y = O.synthetic_batch(og, N, seed=22)
    x32 = np.ascontiguousarray(x, np.float32)
    tr = rp.DecoupledTrainer(_geo(og), 2, rp.PENALTY, rp.SQUARED_L2, N, params=p32)
    loss, acc = tr.evaluate(x32, y)
    logits = O.net_forward(net, x32.astype(np.float64), 0, og.blocks).logits
    want_loss, _ = O.loss_phi(logits, y)
    assert abs(loss - want_loss) <= FP32_TOL * abs(want_loss), (loss, want_loss)
    # per-row argmax from the device logits through the eval kernel
    got_logits = tr.forward(x32)
    dev = torch.from_numpy(got_logits).cuda()
    yd = torch.from_numpy(y.astype(np.int32)).cuda()
    pred = torch.full((N,), -1, dtype=torch.int32, device="cuda")
    wsb = lib().rp_op_eval_workspace_bytes(N)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    l2, hits = C.c_double(), C.c_int64()
    rp.check(lib().rp_op_eval_loss_accuracy(C.c_void_p(dev.data_ptr()), C.c_void_p(yd.data_ptr()), N, og.classes,
                                            C.byref(l2), C.byref(hits), C.c_void_p(pred.data_ptr()),
                                            C.c_void_p(ws.data_ptr()), wsb, None))
    assert l2.value == loss and hits.value == round(acc * N)
    srt = np.sort(logits, axis=1)
    margin = srt[:, -1] - srt[:, -2]
    bound = 1e-4 * np.abs(logits).max()
    sure = margin > bound
    assert sure.mean() > 0.9
    want_pred = O.argmax_lowest(logits)
    assert np.array_equal(pred.cpu().numpy()[sure], want_pred[sure])
    assert hits.value == int((pred.cpu().numpy() == y).sum())
    assert abs(acc - float((want_pred == y).mean())) <= (~sure).sum() / N


def test_argmax_ties_go_to_the_lowest_class():
    """accuracy's strict '>' scan (network.cpp:227-231): all-equal logits predict class 0."""
    N, classes = 37, 10
    logits = torch.zeros(N, classes, device="cuda")
    logits[5, 3] = 1.0
    logits[6, 7] = logits[6, 2] = 2.0     # tie between 2 and 7 -> 2
    y = torch.zeros(N, dtype=torch.int32, device="cuda")
    pred = torch.full((N,), -1, dtype=torch.int32, device="cuda")
    wsb = lib().rp_op_eval_workspace_bytes(N)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    loss, hits = C.c_double(), C.c_int64()
    rp.check(lib().rp_op_eval_loss_accuracy(C.c_void_p(logits.data_ptr()), C.c_void_p(y.data_ptr()), N, classes,
                                            C.byref(loss), C.byref(hits), C.c_void_p(pred.data_ptr()),
                                            C.c_void_p(ws.data_ptr()), wsb, None))
    p = pred.cpu().numpy()
    assert p[5] == 3 and p[6] == 2 and (np.delete(p, [5, 6]) == 0).all()
    assert hits.value == N - 2
    assert abs(loss.value - float(O.loss_phi(logits.double().cpu().numpy(), np.zeros(N, np.int64))[0])) <= 1e-12


@pytest.mark.parametrize("kind", [0, 1, 2])
def test_psi_and_grads_vs_reference_golden(kind):
    """rp_op_psi / rp_op_psi_grad against ref_psi.npz (made by the compiled reference):
    the KATs lambda = [1, 2], x = 0 and the random case with a zero difference (sign0) and
    an exact L-inf tie (first flat index wins)."""
    f = load("ref_psi")
    red = torch.empty(lib().rp_op_reduce_workspace_bytes(), dtype=torch.uint8, device="cuda")
    for lam, x, want_v, want_g in ((np.array([[1.0, 2.0]]), np.zeros((1, 2)), f[f"kat_psi_{kind}"],
                                    f[f"kat_dl_{kind}"]), (f["a"], f["b"], f[f"psi_{kind}"], f[f"dl_{kind}"])):
        tl = torch.from_numpy(lam.astype(np.float32).reshape(-1)).cuda()
        tx = torch.from_numpy(x.astype(np.float32).reshape(-1)).cuda()
        v = C.c_double()
        rp.check(lib().rp_op_psi(kind, C.c_void_p(tl.data_ptr()), C.c_void_p(tx.data_ptr()), tl.numel(), C.byref(v),
                                 C.c_void_p(red.data_ptr()), None))
        assert abs(v.value - float(want_v)) <= 1e-6 * max(1.0, abs(float(want_v))), (kind, v.value, want_v)
        out = torch.full((tl.numel(),), float("nan"), device="cuda")
        rp.check(lib().rp_op_psi_grad(kind, C.c_void_p(tl.data_ptr()), C.c_void_p(tx.data_ptr()), tl.numel(), 1.0,
                                      C.c_void_p(out.data_ptr()), C.c_void_p(red.data_ptr()), None))
        torch.cuda.synchronize()
        got, want = out.cpu().numpy().astype(np.float64), np.asarray(want_g, np.float64).reshape(-1)
        if kind == 0:   # 2 (lambda - x): the fp32 difference rounds once
            assert np.all(np.abs(got - want) <= np.spacing(np.abs(want).astype(np.float32)))
        else:           # sign0 / the L-inf unit mass: exact
            np.testing.assert_array_equal(got, want)
