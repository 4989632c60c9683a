"""Per-unit timestamps of the tcgen05 conv kernel (CTA 0 and 1) for pipeline analysis."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
L = C.CDLL(rp._lib.LIB_PATH)
tr = torch.zeros(2 * 64 * 8, dtype=torch.int64, device="cuda")
n, h, w, c = 256, 32, 32, 64
x = torch.randn(n, h, w, c, device="cuda"); out = torch.empty_like(x)
wt = torch.randn(3, 3, c, c, device="cuda") * 0.05; b = torch.zeros(c, device="cuda")
wsb = lib().rp_op_conv3x3_workspace_bytes(c, c); ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
P = C.c_void_p
xp = torch.empty(2 * x.numel(), dtype=torch.bfloat16, device="cuda")
op = torch.empty_like(xp)
rp.check(lib().rp_op_split_planes(P(x.data_ptr()), x.numel(), P(xp.data_ptr()), P(xp.data_ptr() + 2 * x.numel()), None))
for math in sys.argv[1:] or ("planes", "fp32"):
    sys.stdout.flush()
    for it in range(3):
        if it == 2:
            L.rp_debug_set_trace(P(tr.data_ptr()))
        if math == "planes":
            rp.check(lib().rp_op_conv3x3_planes(n, h, w, c, c, P(xp.data_ptr()), P(wt.data_ptr()), 0, P(b.data_ptr()),
                                                None, 1.0, 1, P(out.data_ptr()), P(op.data_ptr()), P(ws.data_ptr()),
                                                wsb, None))
        else:
            rp.check(lib().rp_op_conv3x3(n, h, w, c, c, P(x.data_ptr()), P(wt.data_ptr()), 0, P(b.data_ptr()), None,
                                         1.0, 1, P(out.data_ptr()), rp.MATH[math], P(ws.data_ptr()), wsb, None))
        torch.cuda.synchronize()
    L.rp_debug_set_trace(None)
    t = tr.cpu().numpy().reshape(2, 64, 8)
    t0 = t[0, 0, 0]
    print(math)
    for cta in range(2):
        for u in range(8):
            row = t[cta, u]
            if row[0] == 0:
                break
            print(f" cta{cta} u{u}: mma_start {(row[0]-t0)/1e3:7.2f} halo_c0 {(row[4]-t0)/1e3:7.2f}"
                  f" mma_end {(row[1]-t0)/1e3:7.2f} epi_start {(row[2]-t0)/1e3:7.2f} epi_end {(row[3]-t0)/1e3:7.2f}"
                  f"  wait_halo {row[5]/1965:6.2f}us wait_w {row[6]/1965:6.2f}us"
                  f"  issue {row[7]:6d} cyc = {row[7] / max(1, row[1] - row[0]):5.3f} GHz")
    tr.zero_()
