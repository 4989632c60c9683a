"""Times the bf16 tape block ops at the C5 shape (N=1024, 32x32, C=256): forward (2 convs),
backward (2 dgrad convs + 2 weight gradients), and the weight gradients alone."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib

n, hw, c = int(sys.argv[1]) if len(sys.argv) > 1 else 1024, 32, 256
dev = torch.device("cuda")
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
geo = rp.Geometry(3, hw, hw, c, c, 2, 10).c()
npar = lib().rp_param_count(C.byref(geo))
tp = (torch.rand(npar, device=dev) - 0.5) * 0.05
off = 9 * 3 * c + c
pb = C.c_void_p(tp.data_ptr() + 4 * off)
ne = n * hw * hw * c
x = (torch.rand(ne, device=dev) - 0.5) * 2
x16 = x.to(torch.bfloat16)
a16, d16, xn16 = (torch.empty(ne, dtype=torch.bfloat16, device=dev) for _ in range(3))
xn = torch.empty(ne, device=dev)
g = (torch.rand(ne, device=dev) - 0.5) * 1e-3
g16 = g.to(torch.bfloat16)
dpre16 = torch.empty(ne, dtype=torch.bfloat16, device=dev)
gb = torch.zeros_like(tp)
wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, rp.MATH["bf16"])
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
fl = 2 * 9 * c * c * n * hw * hw


def timeit(fn, it=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it


tf = timeit(lambda: rp.check(lib().rp_op_block_fwd_bf16t(C.byref(geo), n, P(x), P(x16), pb, P(a16), P(d16), P(xn), P(xn16), P(ws), wsb, None)))
tb = timeit(lambda: rp.check(lib().rp_op_block_bwd_bf16t(C.byref(geo), n, P(x16), P(a16), P(d16), pb, P(g), P(g16), P(dpre16), C.c_void_p(gb.data_ptr() + 4 * off), P(ws), wsb, None)))
wsw = lib().rp_op_conv3x3_wgrad_bf16p_workspace_bytes(n, hw, hw, c, c)
gw = torch.empty(9 * c * c, device=dev)
gbb = torch.empty(c, device=dev)
tw = timeit(lambda: rp.check(lib().rp_op_conv3x3_wgrad_bf16p(n, hw, hw, c, c, P(x16), P(g16), 1.0, P(gw), P(gbb), P(ws), wsw, None)))
print(f"fwd (2 convs) {tf:.3f} ms = {2 * fl / tf / 1e9:.0f} TF; bwd (2 dgrad + 2 wgrad) {tb:.3f} ms; "
      f"wgrad {tw:.3f} ms = {fl / tw / 1e9:.0f} TF; dgrads {tb - 2 * tw:.3f} ms = {2 * fl / (tb - 2 * tw) / 1e9:.0f} TF")
