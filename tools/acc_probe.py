"""Where does the plane conv's error come from?  fprop of one 3x3 conv on the plane path with
the operands optionally pre-rounded so that their low planes vanish (x 2^7 and W 2^8 exact in
fp16): error vs fp64 of the same (rounded) operands, for Ci = 16 .. 256."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
from oracle import respar_oracle as O

def r16(v, s):
    return (np.asarray(v * s, np.float32).astype(np.float16).astype(np.float64) / s).astype(np.float32)

dev = torch.device("cuda")
for ci in (16, 64, 256):
    n, hh, ww, co = 2, 16, 16, 64
    rng = np.random.default_rng(1)
    x0 = rng.uniform(-1, 1, (n, hh, ww, ci)).astype(np.float32)
    w0 = (rng.uniform(-1, 1, (3, 3, ci, co)) / np.sqrt(9 * ci)).astype(np.float32)
    for rx in (False, True):
        for rw in (False, True):
            x = r16(x0, 128.0) if rx else x0
            w = r16(w0, 256.0) if rw else w0
            want = O.conv3x3(x.astype(np.float64), w.astype(np.float64))
            tx, tw = torch.from_numpy(x).to(dev), torch.from_numpy(w).to(dev)
            xp = torch.empty(2 * tx.numel(), dtype=torch.float16, device=dev)
            rp.check(lib().rp_op_split_planes(C.c_void_p(tx.data_ptr()), tx.numel(), C.c_void_p(xp.data_ptr()),
                                              C.c_void_p(xp.data_ptr() + 2 * tx.numel()), None, None))
            out = torch.empty((n, hh, ww, co), device=dev)
            wsb = lib().rp_op_conv3x3_workspace_bytes(ci, co)
            ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
            rp.check(lib().rp_op_conv3x3_planes(n, hh, ww, ci, co, C.c_void_p(xp.data_ptr()), C.c_void_p(tw.data_ptr()),
                                                0, None, None, 1.0, 5, C.c_void_p(out.data_ptr()), None, None, None,
                                                C.c_void_p(ws.data_ptr()), wsb, None))
            torch.cuda.synchronize()
            got = out.cpu().numpy().astype(np.float64)
            err = np.abs(got - want).max() / np.abs(want).max()
            mean_err = (got - want).mean() / np.abs(want).max()
            print(f"ci={ci:3d} x_lo={'0' if rx else 'y'} w_lo={'0' if rw else 'y'}: max rel {err:.2e}  mean (bias) {mean_err:+.2e}",
                  flush=True)
