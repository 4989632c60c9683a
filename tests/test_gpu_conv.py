"""GPU: the 3x3 conv kernels (tcgen05 3xTF32 / TF32 and SIMT) through rp_op_conv3x3,
against the fp64 oracle convolution (oracle/respar_oracle.py conv3x3 / conv3x3_dgrad)
with every fused epilogue."""
import ctypes as C

import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
from oracle import respar_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

EPIS = {0: "bias", 1: "bias_tanh", 2: "resid", 3: "tanh_bwd", 4: "add", 5: "scale"}


def want_epi(epi, acc, bias, aux, h):
    if epi == 0:
        return acc + bias
    if epi == 1:
        return np.tanh(acc + bias)
    if epi == 2:
        return aux + h * (acc + bias)
    if epi == 3:
        return (h * acc) * (1.0 - aux * aux)
    if epi == 4:
        return aux + acc
    return h * acc


def run_conv(n, hh, ww, ci, co, epi, math, dgrad, seed=0, hstep=0.7):
    rng = np.random.default_rng(seed)
    cin, cout = (co, ci) if dgrad else (ci, co)       # dgrad: input has the fwd co channels
    x = rng.uniform(-1, 1, (n, hh, ww, cin)).astype(np.float32)
    w = (rng.uniform(-1, 1, (3, 3, ci, co)) / np.sqrt(9 * ci)).astype(np.float32)
    bias = rng.uniform(-0.2, 0.2, cout).astype(np.float32)
    aux = rng.uniform(-0.9, 0.9, (n, hh, ww, cout)).astype(np.float32)
    acc = O.conv3x3_dgrad(x.astype(np.float64), w.astype(np.float64)) if dgrad else \
        O.conv3x3(x.astype(np.float64), w.astype(np.float64))
    want = want_epi(epi, acc, bias.astype(np.float64), aux.astype(np.float64), np.float32(hstep))
    dev = torch.device("cuda")
    tx, tw, tb = (torch.from_numpy(v).to(dev) for v in (x, w, bias))
    taux = torch.from_numpy(aux).to(dev)
    out = taux.clone() if epi == 4 else torch.empty((n, hh, ww, cout), device=dev)
    wsb = lib().rp_op_conv3x3_workspace_bytes(ci, co)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    use_aux = epi in (2, 3, 4)
    rc = lib().rp_op_conv3x3(n, hh, ww, cin, cout, C.c_void_p(tx.data_ptr()), C.c_void_p(tw.data_ptr()),
                             1 if dgrad else 0, C.c_void_p(tb.data_ptr()),
                             C.c_void_p(out.data_ptr() if epi == 4 else taux.data_ptr()) if use_aux else None,
                             hstep, epi, C.c_void_p(out.data_ptr()), rp.MATH[math], C.c_void_p(ws.data_ptr()),
                             wsb, None)
    rp.check(rc)
    torch.cuda.synchronize()
    return out.cpu().numpy().astype(np.float64), want


SHAPES = [(2, 32, 32, 64, 64), (3, 8, 8, 16, 16), (1, 12, 12, 16, 32), (2, 6, 9, 32, 16), (1, 32, 32, 64, 128),
          (5, 7, 7, 48, 64),
          # wide channels (C5 uses C = 256): several 64-channel output blocks per launch
          (2, 16, 16, 128, 128), (1, 16, 16, 256, 256), (2, 8, 8, 64, 192), (1, 9, 11, 256, 64)]


# 3xTF32 keeps ~21 of fp32's 24 mantissa bits per product: a few 1e-6 relative at K = 576
@pytest.mark.parametrize("math,tol", [("fp32", 2e-5), ("simt", 4e-6), ("tf32", 5e-3)])
@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("dgrad", [False, True])
def test_conv_all_epilogues(shape, math, tol, dgrad):
    n, hh, ww, ci, co = shape
    for epi in range(6):
        got, want = run_conv(n, hh, ww, ci, co, epi, math, dgrad, seed=epi)
        err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-30)
        print(f"{shape} dgrad={dgrad} {math} {EPIS[epi]}: {err:.2e}")
        assert err <= tol, (EPIS[epi], err)


PLANE_SHAPES = [(2, 32, 32, 64, 64), (1, 32, 32, 64, 128), (2, 32, 32, 128, 64), (5, 7, 7, 48, 64),
                (1, 12, 10, 16, 64), (2, 16, 16, 128, 128), (1, 16, 16, 256, 256), (1, 9, 11, 256, 64),
                # the positions-as-M kernel's own shapes (Co in {16, 32}; config C1 is 16 x 28 x 28)
                (3, 28, 28, 16, 16), (2, 9, 13, 32, 16), (1, 6, 7, 16, 32), (2, 17, 5, 32, 32), (1, 1, 1, 16, 16)]


@pytest.fixture(params=["pm", "tc"])
def plane_kernel(request):
    """run the plane convs on conv_pm.cu (positions as M) or conv_tc.cu (channels as M)"""
    lib().rp_op_set_plane_conv_kernel(1 if request.param == "pm" else 0)
    yield request.param
    lib().rp_op_set_plane_conv_kernel(-1)


# plane mode: the input enters as an fp16 pair (22 bits, planes.cuh), W as [W0; W1] (W 2^8, 22 bits);
# dgrad runs on a cotangent-sized input (1e-5) whose pair carries a device scale (in and out)
@pytest.mark.parametrize("shape", PLANE_SHAPES)
@pytest.mark.parametrize("dgrad", [False, True])
def test_conv_planes(shape, dgrad, plane_kernel):
    n, hh, ww, ci, co = shape
    cin, cout = (co, ci) if dgrad else (ci, co)
    which = lib().rp_op_plane_conv_kernel(n, hh, ww, cin, cout)
    if which < 0 or which != (1 if plane_kernel == "pm" else 0):
        pytest.skip(f"{plane_kernel} does not take Ci {cin} -> Co {cout}")
    dev = torch.device("cuda")
    for epi in range(6):
        rng = np.random.default_rng(epi)
        cin, cout = (co, ci) if dgrad else (ci, co)
        x = (rng.uniform(-1, 1, (n, hh, ww, cin)) * (1e-5 if dgrad else 1.0)).astype(np.float32)
        w = (rng.uniform(-1, 1, (3, 3, ci, co)) / np.sqrt(9 * ci)).astype(np.float32)
        bias = (rng.uniform(-0.2, 0.2, cout) * (1e-5 if dgrad else 1.0)).astype(np.float32)
        aux = rng.uniform(-0.9, 0.9, (n, hh, ww, cout)).astype(np.float32)
        if dgrad and epi in (2, 4):
            aux *= 1e-5   # the residual adds a cotangent of the same size
        acc = O.conv3x3_dgrad(x.astype(np.float64), w.astype(np.float64)) if dgrad else \
            O.conv3x3(x.astype(np.float64), w.astype(np.float64))
        want = want_epi(epi, acc, bias.astype(np.float64), aux.astype(np.float64), np.float32(0.7))
        tx, tw, tb, taux = (torch.from_numpy(v).to(dev) for v in (x, w, bias, aux))
        xp = torch.empty(2 * tx.numel(), dtype=torch.float16, device=dev)
        sc = torch.zeros(lib().rp_op_plane_scale_bytes() // 4, device=dev) if dgrad else None
        rp.check(lib().rp_op_split_planes(C.c_void_p(tx.data_ptr()), tx.numel(), C.c_void_p(xp.data_ptr()),
                                          C.c_void_p(xp.data_ptr() + 2 * tx.numel()),
                                          C.c_void_p(sc.data_ptr()) if dgrad else None, None))
        out = taux.clone() if epi == 4 else torch.empty((n, hh, ww, cout), device=dev)
        op = torch.empty(2 * out.numel(), dtype=torch.float16, device=dev)
        wsb = lib().rp_op_conv3x3_workspace_bytes(ci, co)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        use_aux = epi in (2, 3, 4)
        rp.check(lib().rp_op_conv3x3_planes(
            n, hh, ww, cin, cout, C.c_void_p(xp.data_ptr()), C.c_void_p(tw.data_ptr()), 1 if dgrad else 0,
            C.c_void_p(tb.data_ptr()), C.c_void_p(out.data_ptr() if epi == 4 else taux.data_ptr()) if use_aux else None,
            0.7, epi, C.c_void_p(out.data_ptr()), C.c_void_p(op.data_ptr()),
            C.c_void_p(sc.data_ptr()) if dgrad else None, C.c_void_p(sc.data_ptr()) if dgrad else None,
            C.c_void_p(ws.data_ptr()), wsb, None))
        torch.cuda.synchronize()
        got = out.cpu().numpy().astype(np.float64)
        err = np.abs(got - want).max() / max(np.abs(want).max(), 1e-30)
        print(f"planes {shape} dgrad={dgrad} {EPIS[epi]}: {err:.2e}")
        # tcgen05's fp32 accumulation loses ~2^-24 relative per MMA step: the error grows with
        # the reduction length 9 Ci (measured 2e-6 at Ci = 64, 6e-6 at 256; tools/acc_probe.py)
        assert err <= 3e-6 * max(1.0, cin / 64), (EPIS[epi], err)
        s_out = float(sc[0].item()) if dgrad else 128.0   # dgrad: the cotangent's scale; fprop: 2^7
        pl = op.float().cpu().numpy().astype(np.float64)
        rec = (pl[:out.numel()] + pl[out.numel():]).reshape(got.shape) / s_out
        assert np.all(np.abs(rec - got) <= 2.0 ** -22 * np.abs(got) + 2.0 ** -25 / s_out), EPIS[epi]


@pytest.mark.parametrize("shape", [(2, 9, 11, 16, 16), (2, 8, 8, 64, 64)], ids=["co16", "co64"])
def test_conv_planes_16byte_views(shape):
    """conv_pm's epilogue moves whole 32-byte sectors per thread where it can (every access at
    Co < 64, the plane stores at Co = 64); C-ABI callers may pass views that are only 16-byte
    aligned, which must take the exchange-row path for that operand and give the same bits."""
    n, hh, ww, ci, co = shape
    if lib().rp_op_plane_conv_kernel(n, hh, ww, ci, co) != 1:
        pytest.skip("conv_pm does not take this shape")
    dev = torch.device("cuda")
    rng = np.random.default_rng(7)
    x = rng.uniform(-1, 1, (n, hh, ww, ci)).astype(np.float32)
    w = (rng.uniform(-1, 1, (3, 3, ci, co)) / np.sqrt(9 * ci)).astype(np.float32)
    bias = rng.uniform(-0.2, 0.2, co).astype(np.float32)
    aux = rng.uniform(-0.9, 0.9, (n, hh, ww, co)).astype(np.float32)
    tx, tw, tb = (torch.from_numpy(v).to(dev) for v in (x, w, bias))
    xp = torch.empty(2 * tx.numel(), dtype=torch.float16, device=dev)
    rp.check(lib().rp_op_split_planes(C.c_void_p(tx.data_ptr()), tx.numel(), C.c_void_p(xp.data_ptr()),
                                      C.c_void_p(xp.data_ptr() + 2 * tx.numel()), None, None))
    ne = n * hh * ww * co
    wsb = lib().rp_op_conv3x3_workspace_bytes(ci, co)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    res = {}
    for shift in (0, 1):   # 0: 32-byte aligned buffers; 1: every output / aux view 16 bytes off
        taux = torch.empty(ne + 4, device=dev)[4 * shift:4 * shift + ne]
        taux.copy_(torch.from_numpy(aux.ravel()).to(dev))
        out = torch.empty(ne + 4, device=dev)[4 * shift:4 * shift + ne]
        op = torch.empty(2 * ne + 8, dtype=torch.float16, device=dev)[8 * shift:8 * shift + 2 * ne]
        assert (out.data_ptr() % 32 == 16) == bool(shift) and (op.data_ptr() % 32 == 16) == bool(shift)
        rp.check(lib().rp_op_conv3x3_planes(
            n, hh, ww, ci, co, C.c_void_p(xp.data_ptr()), C.c_void_p(tw.data_ptr()), 0, C.c_void_p(tb.data_ptr()),
            C.c_void_p(taux.data_ptr()), 0.7, 2, C.c_void_p(out.data_ptr()), C.c_void_p(op.data_ptr()), None, None,
            C.c_void_p(ws.data_ptr()), wsb, None))
        torch.cuda.synchronize()
        res[shift] = (out.cpu().numpy().copy(), op.cpu().numpy().copy())
    assert np.array_equal(res[0][0], res[1][0]) and np.array_equal(res[0][1], res[1][1])
    acc = O.conv3x3(x.astype(np.float64), w.astype(np.float64))
    want = want_epi(2, acc, bias.astype(np.float64), aux.astype(np.float64), np.float32(0.7))
    got = res[1][0].reshape(want.shape).astype(np.float64)
    assert np.abs(got - want).max() / np.abs(want).max() <= 3e-6


BF16_SHAPES = [(2, 16, 16, 128, 128), (1, 16, 16, 256, 256), (2, 9, 11, 64, 128), (1, 32, 32, 128, 256),
               (2, 8, 8, 64, 64)]   # the last falls back to 3xTF32 (Co % 128 != 0)


# bf16 operands (8-bit mantissa), fp32 accumulation: ~2^-9 relative per product
@pytest.mark.parametrize("shape", BF16_SHAPES)
@pytest.mark.parametrize("dgrad", [False, True])
@pytest.mark.parametrize("epi", [1, 2, 3, 4])
def test_conv_bf16(shape, dgrad, epi):
    n, hh, ww, ci, co = shape
    got, want = run_conv(n, hh, ww, ci, co, epi, "bf16", dgrad, seed=3)
    err = np.abs(got - want).max() / np.abs(want).max()
    print(f"bf16 {shape} dgrad={dgrad} {EPIS[epi]}: {err:.2e}")
    assert err <= 1e-2, err


def test_conv_tc_is_deterministic_and_batch_independent():
    """Per-pixel results do not depend on which other samples share the launch (the
    property reset_lambda_from_forward's chunked forward relies on)."""
    a, _ = run_conv(4, 32, 32, 64, 64, 1, "fp32", False, seed=3)
    b, _ = run_conv(4, 32, 32, 64, 64, 1, "fp32", False, seed=3)
    assert np.array_equal(a, b)


def run_wgrad(n, hh, ww, ci, co, math, seed=0, scale=0.8):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (n, hh, ww, ci)).astype(np.float32)
    g = rng.uniform(-1, 1, (n, hh, ww, co)).astype(np.float32)
    want_w = scale * O.conv3x3_wgrad(x.astype(np.float64), g.astype(np.float64))
    want_b = scale * g.astype(np.float64).reshape(-1, co).sum(axis=0)
    dev = torch.device("cuda")
    tx, tg = torch.from_numpy(x).to(dev), torch.from_numpy(g).to(dev)
    gw = torch.full((3, 3, ci, co), float("nan"), device=dev)
    gb = torch.full((co,), float("nan"), device=dev)
    wsb = lib().rp_op_conv3x3_wgrad_workspace_bytes(n, hh, ww, ci, co)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    rp.check(lib().rp_op_conv3x3_wgrad(n, hh, ww, ci, co, C.c_void_p(tx.data_ptr()), C.c_void_p(tg.data_ptr()),
                                       scale, C.c_void_p(gw.data_ptr()), C.c_void_p(gb.data_ptr()), rp.MATH[math],
                                       C.c_void_p(ws.data_ptr()), wsb, None))
    torch.cuda.synchronize()
    return gw.cpu().numpy().astype(np.float64), gb.cpu().numpy().astype(np.float64), want_w, want_b


WG_SHAPES = [(2, 32, 32, 64, 64), (3, 8, 8, 16, 64), (4, 16, 16, 32, 64), (1, 12, 10, 64, 64), (2, 32, 32, 64, 128),
             (3, 7, 7, 16, 16),
             # ci / co blocks (C5: 256 x 256)
             (2, 16, 16, 128, 128), (1, 16, 16, 256, 256), (2, 8, 8, 192, 64), (2, 8, 8, 64, 256),
             (2, 8, 8, 32, 128)]


@pytest.mark.parametrize("math,tol", [("fp32", 2e-5), ("simt", 4e-6), ("tf32", 5e-3)])
@pytest.mark.parametrize("shape", WG_SHAPES)
def test_wgrad(shape, math, tol):
    gw, gb, ww_, wb = run_wgrad(*shape, math=math)
    ew = np.abs(gw - ww_).max() / np.abs(ww_).max()
    eb = np.abs(gb - wb).max() / np.abs(wb).max()
    print(f"wgrad {shape} {math}: w {ew:.2e} b {eb:.2e}")
    assert ew <= tol and eb <= max(tol, 1e-6), (ew, eb)


@pytest.mark.parametrize("shape", [(2, 16, 16, 128, 128), (1, 16, 16, 256, 256), (2, 8, 8, 128, 256),
                                   (2, 8, 8, 256, 128), (3, 7, 9, 128, 128)])
def test_wgrad_bf16(shape):
    gw, gb, ww_, wb = run_wgrad(*shape, math="bf16")
    ew = np.abs(gw - ww_).max() / np.abs(ww_).max()
    eb = np.abs(gb - wb).max() / np.abs(wb).max()
    print(f"wgrad bf16 {shape}: w {ew:.2e} b {eb:.2e}")
    assert ew <= 1e-2 and eb <= 1e-5, (ew, eb)     # bf16 operands; the bias sums fp32 values


def run_wgrad_planes(n, hh, ww, ci, co, seed=0, scale=0.37):
    rng = np.random.default_rng(seed)
    x = rng.uniform(-1, 1, (n, hh, ww, ci)).astype(np.float32)
    g = (rng.uniform(-1, 1, (n, hh, ww, co)) * 3e-6).astype(np.float32)   # cotangent-sized: a scaled pair
    want_w = scale * O.conv3x3_wgrad(x.astype(np.float64), g.astype(np.float64))
    want_b = scale * g.astype(np.float64).reshape(-1, co).sum(axis=0)
    dev = torch.device("cuda")
    tx, tg = torch.from_numpy(x).to(dev), torch.from_numpy(g).to(dev)
    planes = [torch.empty(t.numel(), dtype=torch.float16, device=dev) for t in (tx, tx, tg, tg)]
    sc = torch.zeros(lib().rp_op_plane_scale_bytes() // 4, device=dev)
    rp.check(lib().rp_op_split_planes(C.c_void_p(tx.data_ptr()), tx.numel(), C.c_void_p(planes[0].data_ptr()),
                                      C.c_void_p(planes[1].data_ptr()), None, None))
    rp.check(lib().rp_op_split_planes(C.c_void_p(tg.data_ptr()), tg.numel(), C.c_void_p(planes[2].data_ptr()),
                                      C.c_void_p(planes[3].data_ptr()), C.c_void_p(sc.data_ptr()), None))
    gw = torch.full((3, 3, ci, co), float("nan"), device=dev)
    gb = torch.full((co,), float("nan"), device=dev)
    wsb = lib().rp_op_conv3x3_wgrad_planes_workspace_bytes(n, hh, ww, ci, co)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    rp.check(lib().rp_op_conv3x3_wgrad_planes(n, hh, ww, ci, co, *[C.c_void_p(t.data_ptr()) for t in planes], scale,
                                              C.c_void_p(sc.data_ptr()), C.c_void_p(gw.data_ptr()),
                                              C.c_void_p(gb.data_ptr()),
                                              C.c_void_p(ws.data_ptr()), wsb, None))
    torch.cuda.synchronize()
    return gw.cpu().numpy().astype(np.float64), gb.cpu().numpy().astype(np.float64), want_w, want_b


# x, g as fp16 plane pairs (22 bits; g with its device scale): fp32-class products
@pytest.mark.parametrize("shape", [(2, 32, 32, 64, 64), (3, 8, 8, 64, 64), (1, 12, 10, 64, 64), (2, 16, 16, 128, 64),
                                   (2, 8, 8, 64, 128), (1, 16, 16, 256, 256), (2, 7, 9, 64, 64),
                                   # the 16-channel kernel (conv_wgrad_small.cu; config C1 = 128 x 28 x 28 x 16)
                                   (128, 28, 28, 16, 16), (3, 7, 9, 16, 16), (2, 5, 6, 16, 32), (1, 1, 1, 16, 16),
                                   (4, 28, 28, 16, 32), (2, 33, 17, 16, 16)])
def test_wgrad_planes(shape):
    gw, gb, ww_, wb = run_wgrad_planes(*shape)
    ew = np.abs(gw - ww_).max() / np.abs(ww_).max()
    eb = np.abs(gb - wb).max() / np.abs(wb).max()
    print(f"wgrad planes {shape}: w {ew:.2e} b {eb:.2e}")
    assert ew <= 1e-6 and eb <= 1e-6, (ew, eb)


def test_wgrad_deterministic():
    a = run_wgrad(2, 32, 32, 64, 64, "fp32", seed=5)
    b = run_wgrad(2, 32, 32, 64, 64, "fp32", seed=5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    a = run_wgrad_planes(16, 28, 28, 16, 16, seed=5)
    b = run_wgrad_planes(16, 28, 28, 16, 16, seed=5)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# The stem S (Cin -> C 3x3 conv, streaming kernels): forward and weight/bias gradients vs the
# fp64 oracle.  Cin = 4, C = 256 has more (row quad, channel octet) register tiles than the
# wgrad kernel has threads (10 x 32 = 320 > 256): every tile must still be computed.
@pytest.mark.parametrize("cin,c", [(1, 16), (3, 64), (3, 128), (3, 256), (4, 256), (2, 32)])
def test_stem_fwd_and_wgrad(cin, c):
    n, hh, ww = 3, 12, 10
    rng = np.random.default_rng(17)
    geo = rp.Geometry(cin, hh, ww, c, c, 1, 10).c()
    npar = lib().rp_param_count(C.byref(geo))
    params = rng.uniform(-0.3, 0.3, npar).astype(np.float32)
    x = rng.uniform(-1, 1, (n, hh, ww, cin)).astype(np.float32)
    g = rng.uniform(-1, 1, (n, hh, ww, c)).astype(np.float32)
    sw = params[:9 * cin * c].reshape(3, 3, cin, c).astype(np.float64)
    sb = params[9 * cin * c:9 * cin * c + c].astype(np.float64)
    want_out = O.conv3x3(x.astype(np.float64), sw) + sb
    want_gw = O.conv3x3_wgrad(x.astype(np.float64), g.astype(np.float64))
    want_gb = g.astype(np.float64).reshape(-1, c).sum(axis=0)
    dev = torch.device("cuda")
    tp, tx, tg = (torch.from_numpy(v).to(dev) for v in (params, x, g))
    out = torch.empty((n, hh, ww, c), device=dev)
    grads = torch.full_like(tp, float("nan"))
    wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["fp32"])
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    # stale, large values in the shared memory the wgrad kernel reuses must not leak in
    junk = torch.full((1 << 22,), 1e6, device=dev)
    junk.mul_(3.0)
    rp.check(lib().rp_op_stem_fwd(C.byref(geo), n, C.c_void_p(tx.data_ptr()), C.c_void_p(tp.data_ptr()),
                                  C.c_void_p(out.data_ptr()), rp.MATH["fp32"], C.c_void_p(ws.data_ptr()), wsb, None))
    rp.check(lib().rp_op_stem_bwd(C.byref(geo), n, C.c_void_p(tx.data_ptr()), C.c_void_p(tg.data_ptr()),
                                  C.c_void_p(grads.data_ptr()), C.c_void_p(ws.data_ptr()), wsb, None))
    torch.cuda.synchronize()
    o64 = out.cpu().numpy().astype(np.float64)
    gr = grads.cpu().numpy().astype(np.float64)
    ew = np.abs(gr[:9 * cin * c].reshape(3, 3, cin, c) - want_gw).max() / np.abs(want_gw).max()
    eb = np.abs(gr[9 * cin * c:9 * cin * c + c] - want_gb).max() / np.abs(want_gb).max()
    eo = np.abs(o64 - want_out).max() / np.abs(want_out).max()
    print(f"stem cin={cin} c={c}: out {eo:.1e} gw {ew:.1e} gb {eb:.1e}")
    assert eo <= 1e-5 and ew <= 1e-5 and eb <= 1e-5, (eo, ew, eb)


# rp_op_stem_fwd_planes: the stem output plus, in the same pass, the planes of it --
# bitwise what rp_op_stem_fwd followed by rp_op_split_planes gives (W % 4 == 0: the fused
# store; W = 10 / 6: the split after the streaming kernel).
@pytest.mark.parametrize("cin,c,hh,ww,lo", [(3, 64, 8, 12, True), (3, 64, 8, 12, False), (1, 16, 7, 10, True),
                                             (3, 256, 4, 8, False), (2, 32, 5, 6, True)])
def test_stem_fwd_planes_matches_split(cin, c, hh, ww, lo):
    n = 3
    rng = np.random.default_rng(23)
    geo = rp.Geometry(cin, hh, ww, c, c, 1, 10).c()
    npar = lib().rp_param_count(C.byref(geo))
    dev = torch.device("cuda")
    tp = torch.from_numpy(rng.uniform(-0.3, 0.3, npar).astype(np.float32)).to(dev)
    tx = torch.from_numpy(rng.uniform(-1, 1, (n, hh, ww, cin)).astype(np.float32)).to(dev)
    e = n * hh * ww * c
    wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["fp32"])
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    out_ref = torch.empty(e, device=dev)
    rp.check(lib().rp_op_stem_fwd(C.byref(geo), n, C.c_void_p(tx.data_ptr()), C.c_void_p(tp.data_ptr()),
                                  C.c_void_p(out_ref.data_ptr()), rp.MATH["fp32"], C.c_void_p(ws.data_ptr()), wsb,
                                  None))
    want = torch.full((2 * e,), 0x7FFF, dtype=torch.int16, device=dev)
    rp.check(lib().rp_op_split_planes(C.c_void_p(out_ref.data_ptr()), e, C.c_void_p(want.data_ptr()),
                                      C.c_void_p(want.data_ptr() + 2 * e) if lo else None, None, None))
    out = torch.full((e,), float("nan"), device=dev)
    got = torch.full((2 * e,), 0x7FFF, dtype=torch.int16, device=dev)
    rp.check(lib().rp_op_stem_fwd_planes(C.byref(geo), n, C.c_void_p(tx.data_ptr()), C.c_void_p(tp.data_ptr()),
                                         C.c_void_p(out.data_ptr()), C.c_void_p(got.data_ptr()),
                                         C.c_void_p(got.data_ptr() + 2 * e) if lo else None, None))
    torch.cuda.synchronize()
    assert torch.equal(out, out_ref)
    assert torch.equal(got, want)   # the lo plane untouched (sentinel) when p1 is NULL
    if not lo:
        assert bool((got[e:] == 0x7FFF).all())


# rp_op_head_loss_bwd_planes: the head backward plus the cotangent's planes (the scaled fp16
# pair, or the bf16 single plane) -- bitwise rp_op_head_loss_bwd followed by rp_op_split_planes.
@pytest.mark.parametrize("c,lo", [(64, True), (128, False), (256, True)])
def test_head_loss_bwd_planes_matches_split(c, lo):
    n, hh, ww, classes = 5, 8, 8, 10
    rng = np.random.default_rng(29)
    geo = rp.Geometry(3, hh, ww, c, c, 1, classes).c()
    npar = lib().rp_param_count(C.byref(geo))
    dev = torch.device("cuda")
    tp = torch.from_numpy(rng.uniform(-0.3, 0.3, npar).astype(np.float32)).to(dev)
    pt = C.c_void_p(tp.data_ptr() + 4 * (npar - (c * classes + classes)))
    e = n * hh * ww * c
    x_end = torch.from_numpy(rng.uniform(-1, 1, e).astype(np.float32)).to(dev)
    labels = torch.from_numpy(rng.integers(0, classes, n).astype(np.int32)).to(dev)
    pooled = torch.empty(n * c, device=dev)
    logits = torch.empty(n * classes, device=dev)
    rp.check(lib().rp_op_head_fwd(C.byref(geo), n, C.c_void_p(x_end.data_ptr()), pt, C.c_void_p(pooled.data_ptr()),
                                  C.c_void_p(logits.data_ptr()), None))
    wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["fp32"])
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    outs = []
    for fused in (False, True):
        loss = torch.zeros(1, dtype=torch.float64, device=dev)
        gt = torch.full((c * classes + classes,), float("nan"), device=dev)
        g = torch.full((e,), float("nan"), device=dev)
        planes = torch.full((2 * e,), 0x7FFF, dtype=torch.int16, device=dev)
        p0 = C.c_void_p(planes.data_ptr())
        p1 = C.c_void_p(planes.data_ptr() + 2 * e) if lo else None
        sc = torch.zeros(lib().rp_op_plane_scale_bytes() // 4, device=dev)
        scp = C.c_void_p(sc.data_ptr()) if lo else None
        args = (C.byref(geo), n, C.c_void_p(pooled.data_ptr()), C.c_void_p(logits.data_ptr()), pt,
                C.c_void_p(labels.data_ptr()), C.c_void_p(loss.data_ptr()), C.c_void_p(gt.data_ptr()),
                C.c_void_p(g.data_ptr()))
        if fused:
            rp.check(lib().rp_op_head_loss_bwd_planes(*args, p0, p1, scp, C.c_void_p(ws.data_ptr()), wsb, None))
        else:
            rp.check(lib().rp_op_head_loss_bwd(*args, C.c_void_p(ws.data_ptr()), wsb, None))
            rp.check(lib().rp_op_split_planes(C.c_void_p(g.data_ptr()), e, p0, p1, scp, None))
        torch.cuda.synchronize()
        outs.append((loss, gt, g, planes, sc[:1]))
    for a, b in zip(*outs):
        assert torch.equal(a, b)
    assert bool(torch.isfinite(outs[1][2]).all())


_MC_SCRIPT = r"""
import sys
sys.path.insert(0, sys.argv[1])
import numpy as np
from tests.test_gpu_conv import run_wgrad_planes
for shape in ((2, 32, 32, 64, 64), (1, 12, 10, 64, 64), (1, 16, 16, 256, 256)):
    gw, gb, ww_, wb = run_wgrad_planes(*shape)
    ew = np.abs(gw - ww_).max() / np.abs(ww_).max()
    eb = np.abs(gb - wb).max() / np.abs(wb).max()
    assert ew <= 1e-6 and eb <= 1e-6, (shape, ew, eb)
print("ok")
"""


def test_wgrad_planes_contiguous_ranges():
    """RP_WGRAD_MAP=contiguous: the plane wgrad with contiguous CTA ranges per tap group (the
    default is CTA triples: CTA 3 t + r is tap group r of triple t's position range) against the
    fp64 oracle at the default kernel's bar."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _MC_SCRIPT, root], env={**os.environ, "RP_WGRAD_MAP": "contiguous"},
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


def test_wgrad_planes_clustered_multicast():
    """RP_WGRAD_MC=1: the 3-CTA cluster form of the plane wgrad (TMA multicast of the shared g / x
    rows, distributed bias sums) against the fp64 oracle at the same bar as the default kernel."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", _MC_SCRIPT, root], env={**os.environ, "RP_WGRAD_MC": "1"},
                       capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stderr[-2000:]


@pytest.mark.parametrize("env", [{"RP_CONV_PAIR": "0"}, {"RP_CONV_PAIR": "1"},
                                 {"RP_CONV_PAIR": "0", "RP_CONV_HALO_SW": "0"},
                                 {"RP_CONV_PM_DIRECT": "7"}, {"RP_CONV_PM_DIRECT": "0"}],
                         ids=["single", "pair", "halo16", "direct", "exchange"])
def test_conv_planes_cta_pair_and_single(env):
    """conv_pm.cu's forms: CTA pairs (M = 256 MMAs across a cluster of two CTAs, each holding half
    of the filter; the Co = 64 default), single CTAs, the halo in 16-byte interleaved rows instead
    of 32-byte swizzled ones, and the epilogue's global accesses all as per-thread sectors (the Co < 64
    default) or all through the exchange rows (the Co = 64 default mixes them), for every Co, through the
    plane-conv parity test and a block's forward and backward, at the same bars."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_conv.py::test_conv_planes", "tests/test_gpu_block_planes.py", "-k", "pm or block"],
                       env={**os.environ, **env}, capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
