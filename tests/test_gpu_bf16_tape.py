"""GPU: the bf16 tape path of RP_MATH_BF16 (config C5) -- the bf16 conv epilogues write bf16
copies of their outputs and both weight gradients read them by TMA (rp_op_conv3x3_wgrad_bf16p,
rp_op_block_fwd_bf16t / rp_op_block_bwd_bf16t) -- against the fp64 oracle on the same
bf16-rounded operands and against the fp32-staged bf16 block ops."""
import ctypes as C

import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from paper_2009_01462_b200 import _lib
from paper_2009_01462_b200._lib import lib
from oracle import respar_oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _p(t):
    return C.c_void_p(t.data_ptr())


def _bf16_round(a):
    return torch.from_numpy(a).to(torch.bfloat16).to(torch.float64).numpy()


@pytest.mark.parametrize("shape", [(2, 16, 16, 128, 128), (1, 16, 16, 256, 256), (2, 8, 8, 128, 256),
                                   (2, 8, 8, 256, 128), (3, 7, 9, 128, 128), (2, 32, 32, 128, 128)])
def test_wgrad_bf16p(shape):
    n, hh, ww, ci, co = shape
    rng = np.random.default_rng(11)
    scale = 0.6
    x = rng.uniform(-1, 1, (n, hh, ww, ci)).astype(np.float32)
    g = rng.uniform(-1, 1, (n, hh, ww, co)).astype(np.float32)
    xb, gbf = _bf16_round(x), _bf16_round(g)
    # exact bf16 products, fp64 sums: the kernel differs only by its fp32 accumulation
    want_w = scale * O.conv3x3_wgrad(xb, gbf)
    want_b = scale * gbf.reshape(-1, co).sum(axis=0)
    dev = torch.device("cuda")
    x16 = torch.from_numpy(x).to(dev).to(torch.bfloat16)
    g16 = torch.from_numpy(g).to(dev).to(torch.bfloat16)
    gw = torch.full((3, 3, ci, co), float("nan"), device=dev)
    gb = torch.full((co,), float("nan"), device=dev)
    wsb = lib().rp_op_conv3x3_wgrad_bf16p_workspace_bytes(n, hh, ww, ci, co)
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    rp.check(lib().rp_op_conv3x3_wgrad_bf16p(n, hh, ww, ci, co, _p(x16), _p(g16), scale, _p(gw), _p(gb), _p(ws), wsb,
                                             None))
    torch.cuda.synchronize()
    gw64, gb64 = gw.cpu().numpy().astype(np.float64), gb.cpu().numpy().astype(np.float64)
    ew = np.abs(gw64 - want_w).max() / np.abs(want_w).max()
    eb = np.abs(gb64 - want_b).max() / np.abs(want_b).max()
    print(f"wgrad bf16p {shape}: w {ew:.2e} b {eb:.2e}")
    assert ew <= 2e-5 and eb <= 2e-5, (ew, eb)


def test_wgrad_bf16p_rejects_narrow_channels():
    wsb = 1 << 20
    rc = lib().rp_op_conv3x3_wgrad_bf16p(1, 8, 8, 64, 64, C.c_void_p(16), C.c_void_p(16), 1.0, C.c_void_p(16),
                                         None, C.c_void_p(16), wsb, None)
    assert rc == _lib.RP_ERR_SHAPE


def _rel(a, b):
    a = a.double().cpu()
    b = b.double().cpu()
    return float((a - b).abs().max() / b.abs().max())


def test_block_bf16_tape_matches_staged_bf16_block():
    """The tape path feeds every conv the bf16 copy of its input -- the values the staged
    path's converters produce -- so its forward output is bitwise the staged path's; the
    backward differs only through the bf16-rounded tanh derivative (2^-9 relative)."""
    n, hw, c = 2, 16, 128
    geo = rp.Geometry(3, hw, hw, c, c, 2, 10).c()
    assert lib().rp_op_block_bf16_tape_supported(C.byref(geo), n, rp.MATH["bf16"]) == 1
    assert lib().rp_op_block_bf16_tape_supported(C.byref(geo), n, rp.MATH["fp32"]) == 0
    dev = torch.device("cuda")
    gen = torch.Generator(device="cpu").manual_seed(5)
    npar = lib().rp_param_count(C.byref(geo))
    params = (torch.rand(npar, generator=gen) - 0.5) * 0.1
    tp = params.to(dev)
    off = 9 * 3 * c + c      # block 0 (after the stem w, b)
    pb = C.c_void_p(tp.data_ptr() + 4 * off)
    ne = n * hw * hw * c
    tx = ((torch.rand(ne, generator=gen) - 0.5) * 2).to(dev)
    tup = ((torch.rand(ne, generator=gen) - 0.5) * 2).to(dev)
    wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["bf16"])
    ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
    bf = rp.MATH["bf16"]

    a_ref, xn_ref = torch.empty(ne, device=dev), torch.empty(ne, device=dev)
    rp.check(lib().rp_op_block_fwd(C.byref(geo), n, _p(tx), pb, _p(a_ref), _p(xn_ref), bf, _p(ws), wsb, None))
    x16 = tx.to(torch.bfloat16)
    a16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
    d16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
    xn = torch.empty(ne, device=dev)
    xn16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
    rp.check(lib().rp_op_block_fwd_bf16t(C.byref(geo), n, _p(tx), _p(x16), pb, _p(a16), _p(d16), _p(xn), _p(xn16),
                                         _p(ws), wsb, None))
    torch.cuda.synchronize()
    assert torch.equal(a16, a_ref.to(torch.bfloat16))
    assert _rel(d16, (1 - a_ref * a_ref).to(torch.bfloat16)) <= 2 ** -8
    assert torch.equal(xn, xn_ref)
    assert torch.equal(xn16, xn.to(torch.bfloat16))

    g_io = tup.clone()
    g16 = g_io.to(torch.bfloat16)
    dpre16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
    gb = torch.zeros_like(tp)
    rp.check(lib().rp_op_block_bwd_bf16t(C.byref(geo), n, _p(x16), _p(a16), _p(d16), pb, _p(g_io), _p(g16),
                                         _p(dpre16), C.c_void_p(gb.data_ptr() + 4 * off), _p(ws), wsb, None))
    g_ref = tup.clone()
    dpre_ref = torch.empty(ne, device=dev)
    gb_ref = torch.zeros_like(tp)
    rp.check(lib().rp_op_block_bwd(C.byref(geo), n, _p(tx), _p(a_ref), pb, _p(g_ref), _p(dpre_ref),
                                   C.c_void_p(gb_ref.data_ptr() + 4 * off), bf, _p(ws), wsb, None))
    torch.cuda.synchronize()
    e_dpre, e_g = _rel(dpre16, dpre_ref), _rel(g_io, g_ref)
    assert torch.equal(g16, g_io.to(torch.bfloat16))
    L = 9 * c * c
    blk = gb[off:off + 2 * L + 2 * c].cpu().numpy().astype(np.float64)
    ref = gb_ref[off:off + 2 * L + 2 * c].cpu().numpy().astype(np.float64)
    w_idx = np.r_[0:L, L + c:2 * L + c]
    b_idx = np.r_[L:L + c, 2 * L + c:2 * L + 2 * c]
    ew = np.abs(blk[w_idx] - ref[w_idx]).max() / np.abs(ref[w_idx]).max()
    eb = np.abs(blk[b_idx] - ref[b_idx]).max() / np.abs(ref[b_idx]).max()
    print(f"bf16 tape block: dpre {e_dpre:.2e} g {e_g:.2e} gW {ew:.2e} gb {eb:.2e}")
    assert e_dpre <= 1e-2 and e_g <= 1e-2 and ew <= 1e-2 and eb <= 1e-2, (e_dpre, e_g, ew, eb)


def test_bf16_tape_halo_interleave_fallback():
    """RP_BF16_HALO_SW=0: the bf16 tape conv with its halo in 16-byte interleaved rows instead of
    64-byte swizzled ones passes the same block test."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-x", "-m", "gpu", "-p", "no:cacheprovider",
                        "tests/test_gpu_bf16_tape.py::test_block_bf16_tape_matches_staged_bf16_block"],
                       env={**os.environ, "RP_BF16_HALO_SW": "0"}, capture_output=True, text=True, timeout=600,
                       cwd=root)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
