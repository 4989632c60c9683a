"""Times the stem / head kernels at the C2 shape through the C ABI (CUDA events)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
P = C.c_void_p
g = rp.Geometry(3, 32, 32, 64, 64, 16, 10)
n = 256
geo = g.c()
x = torch.randn(n, 32, 32, 3, device="cuda")
x0 = torch.empty(n, 32, 32, 64, device="cuda")
p = torch.randn(rp.param_count(g), device="cuda") * 0.05
gs = torch.zeros_like(p)
wsb = lib().rp_op_workspace_bytes(C.byref(geo), n, 0)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
def t(fn, it=5):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(it): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / it * 1e3
print("stem fwd  %.1f us" % t(lambda: rp.check(lib().rp_op_stem_fwd(C.byref(geo), n, P(x.data_ptr()), P(p.data_ptr()), P(x0.data_ptr()), 0, None, 0, None))))
print("stem wgrad %.1f us" % t(lambda: rp.check(lib().rp_op_stem_bwd(C.byref(geo), n, P(x.data_ptr()), P(x0.data_ptr()), P(gs.data_ptr()), P(ws.data_ptr()), wsb, None))))
