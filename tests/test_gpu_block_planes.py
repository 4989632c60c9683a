"""GPU: the plane-pair residual block (rp_op_block_fwd_planes / rp_op_block_bwd_planes) that
the fp32 trainer runs on tcgen05 shapes, against the fp64 oracle block (block_forward /
block_vjp, network.cpp:82-106) and against the fp32-operand block path.

Every conv of the plane path reads its input as an fp16 plane pair (v s = p0 + p1: 22
significant bits, planes.cuh) and writes the plane pair of its output, which must reconstruct
the fp32 output to fp16-pair precision (|v s - p0 - p1| <= 2^-22 |v s| + 2^-25, the second term
for subnormal low planes).  The cotangent enters at 1e-5 scale (the size of a synthetic-loss
upstream), so its pair carries a device scale.  Tolerances: 1e-5 of the tensor's max |value|
against the fp64 oracle for activations / cotangents, 2e-5 for the weight gradients (the
operands are fp32-class; tcgen05's fp32 accumulation costs ~2e-6 per 576-term conv)."""
import ctypes as C

import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib, rp_geometry
from oracle import respar_oracle as O

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")

GW_TOL = 2e-5    # weight / bias gradients, relative to the tensor's max |value|
FWD_TOL = 1e-5   # a, x_next, input cotangent (tcgen05 fp32 accumulation: ~2e-6 per conv)


def _p(t):
    return C.c_void_p(t.data_ptr())


ACT = 128.0   # the forward activations' plane scale (planes.cuh kActPlaneScale)


def _planes_to_f64(t, n, scale=ACT):
    b = t.view(torch.float16).float().cpu().numpy().astype(np.float64)
    return (b[:n] + b[n:2 * n]) / scale


def _pair_ok(t, n, v, scale=ACT):
    return np.all(np.abs(_planes_to_f64(t, n, scale) - v) <= (2.0 ** -22 * np.abs(v) + 2.0 ** -25 / scale))


def _rel(got, want):
    return np.abs(got - want).max() / max(np.abs(want).max(), 1e-30)


@pytest.mark.parametrize("n,hw,c,ch", [(4, 16, 64, 64), (2, 32, 64, 128), (3, 8, 128, 64),
                                       (8, 28, 16, 16), (3, 9, 16, 16)])   # C1: 16 channels (conv_pm, wgrad_small)
def test_block_planes(n, hw, c, ch):
    og = O.Geometry(in_channels=3, height=hw, width=hw, channels=c, hidden=ch, blocks=1, classes=10,
                    activation=O.TANH, step_h=0.5)
    net = O.make_net(og, O.Rng(11))
    net.b1[0][...] = O.rng_uniform(O.Rng(12), ch, -0.1, 0.1)
    net.b2[0][...] = O.rng_uniform(O.Rng(13), c, -0.1, 0.1)
    flat = net.flat().astype(np.float32)
    net32 = net.astype(np.float32).astype(np.float64)
    geo = rp_geometry(3, hw, hw, c, ch, 1, 10, 0, 0.5)
    assert lib().rp_op_block_planes_supported(C.byref(geo), n, rp.MATH["fp32"]) == 1
    assert lib().rp_op_block_planes_supported(C.byref(geo), n, rp.MATH["bf16"]) == 0

    rng = np.random.default_rng(5)
    x = rng.uniform(-1, 1, (n, hw, hw, c)).astype(np.float32)
    up = (rng.uniform(-1, 1, (n, hw, hw, c)) * 1e-5).astype(np.float32)
    dev = torch.device("cuda")
    tx, tup, tp = (torch.from_numpy(v).to(dev) for v in (x, up, flat))
    off = lib().rp_param_offset_block(C.byref(geo), 0)
    pb = C.c_void_p(tp.data_ptr() + 4 * off)
    wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["fp32"])
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    ne, nh = n * hw * hw * c, n * hw * hw * ch

    # fp32-operand reference path
    a_ref = torch.empty(nh, device=dev)
    xn_ref = torch.empty(ne, device=dev)
    rp.check(lib().rp_op_block_fwd(C.byref(geo), n, _p(tx), pb, _p(a_ref), _p(xn_ref), rp.MATH["fp32"], _p(ws), wsb,
                                   None))
    # plane path
    a = torch.empty(nh, device=dev)
    xn = torch.empty(ne, device=dev)
    a_p = torch.empty(2 * nh, dtype=torch.int16, device=dev)
    xn_p = torch.empty(2 * ne, dtype=torch.int16, device=dev)
    x_p = torch.empty(2 * ne, dtype=torch.int16, device=dev)
    rp.check(lib().rp_op_split_planes(_p(tx), ne, _p(x_p), C.c_void_p(x_p.data_ptr() + 2 * ne), None, None))
    # the block's filters prepared once (rp_op_prep_planes_filters) vs per conv (filters = NULL):
    # bitwise the same
    fbytes = lib().rp_op_planes_filters_bytes(C.byref(geo), 1)
    ffwd = torch.empty(fbytes, dtype=torch.uint8, device=dev)
    fbwd = torch.empty(fbytes, dtype=torch.uint8, device=dev)
    rp.check(lib().rp_op_prep_planes_filters(C.byref(geo), pb, 1, 0, _p(ffwd), None))
    rp.check(lib().rp_op_prep_planes_filters(C.byref(geo), pb, 1, 1, _p(fbwd), None))
    rp.check(lib().rp_op_block_fwd_planes(C.byref(geo), n, _p(tx), _p(x_p), pb, _p(a), _p(xn), _p(a_p), _p(xn_p),
                                          None, _p(ws), wsb, None))
    xn_self = xn.clone()
    rp.check(lib().rp_op_block_fwd_planes(C.byref(geo), n, _p(tx), _p(x_p), pb, _p(a), _p(xn), _p(a_p), _p(xn_p),
                                          _p(ffwd), _p(ws), wsb, None))
    torch.cuda.synchronize()
    assert torch.equal(xn, xn_self)
    a64, xn64 = a.cpu().numpy().astype(np.float64), xn.cpu().numpy().astype(np.float64)
    assert _rel(a64, a_ref.cpu().numpy().astype(np.float64)) < FWD_TOL
    assert _rel(xn64, xn_ref.cpu().numpy().astype(np.float64)) < FWD_TOL
    assert _pair_ok(a_p, nh, a64)
    assert _pair_ok(xn_p, ne, xn64)
    want_xn, cache = O.block_forward(net32, 0, x.astype(np.float64))
    assert _rel(xn64.reshape(want_xn.shape), want_xn) < FWD_TOL

    # backward: plane path vs oracle and vs fp32-operand path
    g_io = tup.clone().reshape(-1)
    g_p = torch.empty(2 * ne, dtype=torch.int16, device=dev)
    gscale = torch.zeros(lib().rp_op_plane_scale_bytes() // 4, device=dev)
    rp.check(lib().rp_op_split_planes(_p(g_io), ne, _p(g_p), C.c_void_p(g_p.data_ptr() + 2 * ne), _p(gscale), None))
    dpre = torch.empty(nh, device=dev)
    dpre_p = torch.empty(2 * nh, dtype=torch.int16, device=dev)
    gb = torch.zeros_like(tp)
    gbp = C.c_void_p(gb.data_ptr() + 4 * off)
    rp.check(lib().rp_op_block_bwd_planes(C.byref(geo), n, _p(x_p), _p(a), _p(a_p), pb, _p(g_io), _p(g_p), _p(gscale),
                                          _p(dpre),
                                          _p(dpre_p), gbp, _p(fbwd), _p(ws), wsb, None))
    g_ref = tup.clone().reshape(-1)
    gb_ref = torch.zeros_like(tp)
    rp.check(lib().rp_op_block_bwd(C.byref(geo), n, _p(tx), _p(a_ref), pb, _p(g_ref), _p(dpre),
                                   C.c_void_p(gb_ref.data_ptr() + 4 * off), rp.MATH["fp32"], _p(ws), wsb, None))
    torch.cuda.synchronize()
    g64 = g_io.cpu().numpy().astype(np.float64)
    assert _rel(g64, g_ref.cpu().numpy().astype(np.float64)) < FWD_TOL
    s = float(gscale[0].item())
    assert s == 2.0 ** (8 - np.frexp(np.abs(up).max())[1])     # max |g s| in [2^7, 2^8)
    assert _pair_ok(g_p, ne, g64, s)

    p_prev, (gw1, gb1, gw2, gb2) = O.block_vjp(net32, 0, O.BlockCache(x.astype(np.float64), a64.reshape(
        n, hw, hw, ch)), up.astype(np.float64))
    assert _rel(g64.reshape(p_prev.shape), p_prev) < FWD_TOL
    got = O.zero_net(og)
    got.load_flat(gb.cpu().numpy().astype(np.float64))
    ref = O.zero_net(og)
    ref.load_flat(gb_ref.cpu().numpy().astype(np.float64))
    for name, want in (("w1", gw1), ("b1", gb1), ("w2", gw2), ("b2", gb2)):
        gv = np.asarray(getattr(got, name)[0])
        rv = np.asarray(getattr(ref, name)[0])
        assert _rel(gv, want) < GW_TOL, name
        assert _rel(gv, rv) < GW_TOL, name
