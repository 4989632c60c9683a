"""Per-epilogue timing of the tcgen05 conv at the C2 block shape (CUDA events)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
P = C.c_void_p
n, h, w, c = 256, 32, 32, 64
x = torch.randn(n, h, w, c, device="cuda"); aux = torch.randn_like(x) * 0.5; out = torch.empty_like(x)
wt = torch.randn(3, 3, c, c, device="cuda") * 0.05; b = torch.zeros(c, device="cuda")
wsb = lib().rp_op_conv3x3_workspace_bytes(c, c); ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
names = {0: "bias", 1: "bias_tanh", 2: "resid", 3: "tanh_bwd", 4: "add", 5: "scale"}
for epi in range(6):
    for dg in (0, 1):
        f = lambda: rp.check(lib().rp_op_conv3x3(n, h, w, c, c, P(x.data_ptr()), P(wt.data_ptr()), dg, P(b.data_ptr()),
                                                 P(aux.data_ptr()), 0.5, epi, P(out.data_ptr()), 0, P(ws.data_ptr()), wsb,
                                                 None))
        f(); torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(5): f()
        e.record(); torch.cuda.synchronize()
        print(f"{'dgrad' if dg else 'fprop'} {names[epi]:10s} {s.elapsed_time(e) / 5 * 1e3:7.1f} us")
