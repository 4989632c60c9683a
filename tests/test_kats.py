"""Known-answer tests of the reference's own suites, on the oracle
(CPU) and -- marked gpu -- on the B200 kernels through the C ABI.

    block identity / W = I         test_network.cpp:61-132
    loss: uniform logits -> ln 3   test_network.cpp:196-225
    multiplier step -> -8e-8       test_decoupled.cpp:309-327
    psi values                     test_penalty.cpp:32-38 (also in test_oracle.py)
"""
import ctypes as C
import math

import numpy as np
import pytest

from oracle import respar_oracle as O


def _dense(d=2, h=2, L=1, classes=3, act=O.TANH):
    return O.Geometry(in_channels=d, height=1, width=1, channels=d, hidden=h, blocks=L, classes=classes,
                      activation=act)


def _identity_block_net(g):
    net = O.zero_net(g)
    net.w1[0][1, 1] = np.eye(g.channels, g.hidden)
    net.w2[0][1, 1] = np.eye(g.hidden, g.channels)
    return net


def test_kat_zero_block_is_identity():
    g = _dense()
    net = O.zero_net(g)
    x = np.array([[0.3, -1.2], [2.0, 0.5]]).reshape(2, 1, 1, 2)
    y, _ = O.block_forward(net, 0, x)
    np.testing.assert_array_equal(y, x)


def test_kat_identity_weights():
    # [[1, 0]] with W1 = W2 = I  ->  [[1 + tanh 1, 0]]
    g = _dense()
    net = _identity_block_net(g)
    x = np.array([[1.0, 0.0]]).reshape(1, 1, 1, 2)
    y, _ = O.block_forward(net, 0, x)
    np.testing.assert_allclose(y.reshape(-1), [1.0 + math.tanh(1.0), 0.0], rtol=0, atol=1e-15)


def test_kat_uniform_logits_loss_is_ln3():
    logits = np.zeros((4, 3))
    loss, grad = O.loss_phi(logits, np.array([0, 1, 2, 1]))
    assert abs(loss - math.log(3.0)) <= 1e-15
    assert np.abs(grad.sum(axis=1)).max() <= 1e-12


def test_kat_multiplier_step():
    # kappa = 0, beta = 0.1, # = 200 x 8 = 1600, lambda - X = 0.01 -> kappa = -8e-8
    g = O.Geometry(in_channels=8, height=1, width=1, channels=8, hidden=8, blocks=2, classes=3)
    net = O.zero_net(g)
    tr = O.DecoupledTrainer(net, 2, O.ALM, O.SQUARED_L2, 200)
    x = np.zeros((200, 1, 1, 8))
    tr.reset_lambda_from_forward(x)
    tr.stage(1).lam[...] = tr.stage(0).boundary_out + 0.01
    tr.correct_multiplier(1, 0.1, 1e-9, 0, 200)
    np.testing.assert_allclose(tr.stage(1).kappa, -8e-8, rtol=1e-12, atol=0)


# ------------------------------------------------------------------ device
@pytest.mark.gpu
def test_kat_device_block_and_loss():
    torch = pytest.importorskip("torch")
    import paper_2009_01462_b200 as rp
    from paper_2009_01462_b200._lib import lib, rp_geometry

    g = _dense()
    net = _identity_block_net(g)
    flat = net.flat().astype(np.float32)
    geo = rp_geometry(g.in_channels, 1, 1, g.channels, g.hidden, g.blocks, g.classes, 0, 1.0)
    n = 1
    x = torch.tensor([[1.0, 0.0]], device="cuda")
    a = torch.empty(n, g.hidden, device="cuda")
    out = torch.empty(n, g.channels, device="cuda")
    p = torch.from_numpy(flat).cuda()
    off = lib().rp_param_offset_block(C.byref(geo), 0)
    wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["fp32"])
    ws = torch.empty(max(wsb, 256), dtype=torch.uint8, device="cuda")
    rp.check(lib().rp_op_block_fwd(C.byref(geo), n, C.c_void_p(x.data_ptr()), C.c_void_p(p.data_ptr() + 4 * off),
                                   C.c_void_p(a.data_ptr()), C.c_void_p(out.data_ptr()), rp.MATH["fp32"],
                                   C.c_void_p(ws.data_ptr()), wsb, None))
    torch.cuda.synchronize()
    np.testing.assert_allclose(out.cpu().numpy().reshape(-1), [1.0 + math.tanh(1.0), 0.0], rtol=2e-7, atol=1e-7)

    # multiplier step on the device trainer: kappa -> -8e-8 (fp32)
    g8 = rp.Geometry(8, 1, 1, 8, 8, 2, 3)
    tr = rp.DecoupledTrainer(g8, 2, rp.ALM, rp.SQUARED_L2, 200, params=np.zeros(rp.param_count(g8), np.float32))
    tr.reset_lambda_from_forward(np.zeros((200, 1, 1, 8), np.float32))
    tr.set_state(1, rp.LAMBDA, tr.state(0, rp.BOUNDARY_OUT) + np.float32(0.01))
    tr.correct_multiplier(1, 0.1, 1e-9, 0, 200)
    np.testing.assert_allclose(tr.state(1, rp.KAPPA), -8e-8, rtol=1e-6, atol=0)
