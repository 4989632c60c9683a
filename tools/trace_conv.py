"""Per-unit timestamps of the tcgen05 plane conv (CTAs 0 and 1): when each unit's MMA issue
starts / ends, when its first halo chunk was ready, when the epilogue drained it; cycles the
MMA warp waited for halo chunks.  Diagnostics only: calls the library's internal trace setter
(rp::k::conv3x3_tc_set_trace) through its C++ symbol.

    python tools/trace_conv.py [fprop|dgrad] ...
"""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
set_trace = getattr(C.CDLL(rp._lib.LIB_PATH), "_ZN2rp1k20conv3x3_tc_set_traceEPy")
set_trace.argtypes = [C.c_void_p]
tr = torch.zeros(2 * 64 * 8, dtype=torch.int64, device="cuda")
n, h, w, c = 256, 32, 32, 64
x = torch.rand(n, h, w, c, device="cuda") * 2 - 1
aux = torch.rand(n, h, w, c, device="cuda") * 2 - 1
out = torch.empty_like(x)
wt = torch.randn(3, 3, c, c, device="cuda") * 0.05
b = torch.zeros(c, device="cuda")
wsb = lib().rp_op_conv3x3_workspace_bytes(c, c)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
P = C.c_void_p
xp = torch.empty(2 * x.numel(), dtype=torch.float16, device="cuda")
op = torch.empty_like(xp)
rp.check(lib().rp_op_split_planes(P(x.data_ptr()), x.numel(), P(xp.data_ptr()), P(xp.data_ptr() + 2 * x.numel()),
                                  None, None))
for which in sys.argv[1:] or ("fprop", "dgrad"):
    d = which == "dgrad"
    for it in range(4):
        if it == 3:
            set_trace(tr.data_ptr())
        rp.check(lib().rp_op_conv3x3_planes(n, h, w, c, c, P(xp.data_ptr()), P(wt.data_ptr()), int(d),
                                            P(b.data_ptr()), P(aux.data_ptr()) if d else None, 1.0, 3 if d else 1,
                                            P(out.data_ptr()), P(op.data_ptr()), None, None, P(ws.data_ptr()), wsb,
                                            None))
        torch.cuda.synchronize()
    set_trace(None)
    t = tr.cpu().numpy().reshape(2, 64, 8)
    t0 = t[0, 0, 0]
    print(which)
    for cta in range(2):
        for u in range(10):
            row = t[cta, u]
            if row[0] == 0:
                break
            print(f" cta{cta} u{u}: mma {(row[0]-t0)/1e3:7.2f} .. {(row[1]-t0)/1e3:7.2f} us (halo c0 {(row[4]-t0)/1e3:7.2f})"
                  f"  epi {(row[2]-t0)/1e3:7.2f} .. {(row[3]-t0)/1e3:7.2f}"
                  f"  wait_halo {row[5]:6d} cyc  issue {row[7]:6d} cyc = {row[7] / max(1, row[1] - row[0]):5.3f} GHz")
    tr.zero_()
