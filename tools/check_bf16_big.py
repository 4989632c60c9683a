"""C5-sized consistency checks of the bf16 tape kernels against the fp32-input bf16 kernels
(same bf16 products): wgrad_bf16p vs wgrad(bf16), conv bf16-input vs fp32-input."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib

n, h, w, c = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 32, 32, 256
dev = torch.device("cuda")
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
x = (torch.rand(n, h, w, c, device=dev) - 0.5) * 2
g = (torch.rand(n, h, w, c, device=dev) - 0.5) * 1e-6
x16, g16 = x.to(torch.bfloat16), g.to(torch.bfloat16)
wsb = max(lib().rp_op_conv3x3_wgrad_workspace_bytes(n, h, w, c, c), lib().rp_op_conv3x3_wgrad_bf16p_workspace_bytes(n, h, w, c, c))
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
gw1, gb1 = torch.empty(3, 3, c, c, device=dev), torch.empty(c, device=dev)
gw2, gb2 = torch.empty(3, 3, c, c, device=dev), torch.empty(c, device=dev)
rp.check(lib().rp_op_conv3x3_wgrad(n, h, w, c, c, P(x), P(g), 1.0, P(gw1), P(gb1), rp.MATH["bf16"], P(ws), wsb, None))
rp.check(lib().rp_op_conv3x3_wgrad_bf16p(n, h, w, c, c, P(x16), P(g16), 1.0, P(gw2), P(gb2), P(ws), wsb, None))
torch.cuda.synchronize()
rel = lambda a, b: float((a - b).abs().max() / b.abs().max())  # noqa: E731
print(f"wgrad n={n}: w rel {rel(gw2, gw1):.2e} (max {gw1.abs().max():.3e} vs {gw2.abs().max():.3e}) b rel {rel(gb2, gb1):.2e}")

# block forward: bf16-input tape path vs fp32-input bf16 path, bitwise; backward with g = 0
geo = rp.Geometry(3, h, w, c, c, 2, 10).c()
npar = lib().rp_param_count(C.byref(geo))
tp = (torch.rand(npar, device=dev) - 0.5) * 0.05
off = 9 * 3 * c + c
pb = C.c_void_p(tp.data_ptr() + 4 * off)
ne = n * h * w * c
wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["bf16"])
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
tx = x.reshape(-1)
a_ref, xn_ref = torch.empty(ne, device=dev), torch.empty(ne, device=dev)
rp.check(lib().rp_op_block_fwd(C.byref(geo), n, P(tx), pb, P(a_ref), P(xn_ref), rp.MATH["bf16"], P(ws), wsb, None))
a16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
d16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
xn = torch.empty(ne, device=dev)
xn16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
rp.check(lib().rp_op_block_fwd_bf16t(C.byref(geo), n, P(tx), P(x16), pb, P(a16), P(d16), P(xn), P(xn16), P(ws), wsb, None))
torch.cuda.synchronize()
print("fwd: a16 == bf16(a_ref):", torch.equal(a16, a_ref.to(torch.bfloat16)), " xn == xn_ref:", torch.equal(xn, xn_ref),
      " max |xn - xn_ref|:", float((xn - xn_ref).abs().max()))
g_io = torch.zeros(ne, device=dev)
gz16 = g_io.to(torch.bfloat16)
dpre16 = torch.full((ne,), 7.0, dtype=torch.bfloat16, device=dev)
gb = torch.zeros_like(tp)
rp.check(lib().rp_op_block_bwd_bf16t(C.byref(geo), n, P(x16), P(a16), P(d16), pb, P(g_io), P(gz16), P(dpre16),
                                     C.c_void_p(gb.data_ptr() + 4 * off), P(ws), wsb, None))
torch.cuda.synchronize()
print("bwd g=0: max |g| after", float(g_io.abs().max()), " max |dpre16|", float(dpre16.float().abs().max()),
      " max |grads|", float(gb.abs().max()), " nonzero g count", int((g_io != 0).sum()))
