"""Per-block timestamps of the tcgen05 wgrad kernel (CTA 0 and 1) for pipeline analysis."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
L = C.CDLL(rp._lib.LIB_PATH)
P = C.c_void_p
tr = torch.zeros(2 * 64 * 8, dtype=torch.int64, device="cuda")
n, h, w, c = int(os.environ.get("TN", 256)), 32, 32, int(os.environ.get("TC", 64))
x = torch.randn(n, h, w, c, device="cuda"); g = torch.randn(n, h, w, c, device="cuda")
gw = torch.empty(3, 3, c, c, device="cuda"); gb = torch.empty(c, device="cuda")
wsb = lib().rp_op_conv3x3_wgrad_workspace_bytes(n, h, w, c, c)
ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
for math in os.environ.get("MATHS", "fp32,tf32").split(","):
    for it in range(3):
        if it == 2:
            L.rp_debug_set_trace(P(tr.data_ptr()))
        rp.check(lib().rp_op_conv3x3_wgrad(n, h, w, c, c, P(x.data_ptr()), P(g.data_ptr()), C.c_double(1.0),
                                           P(gw.data_ptr()), P(gb.data_ptr()), rp.MATH[math], P(ws.data_ptr()),
                                           wsb, None))
        torch.cuda.synchronize()
    L.rp_debug_set_trace(None)
    t = tr.cpu().numpy().reshape(2, 64, 8)
    t0 = t[0, 0, 0]
    print(math, "(us)  tma_issue  conv_in  conv_done  mma_start  mma_issued  first_piece")
    for cta in range(1):
        for b in [0, 1, 2, 3, 30, 31, 62]:
            row = t[cta, b]
            if row[0] == 0:
                continue
            print(f" cta{cta} b{b:2d}: " + " ".join(f"{(v - t0) / 1e3:9.2f}" for v in row[:6]) +
                  f"  piece_wait {row[6] / 1900:7.2f}us")
    tr.zero_()
