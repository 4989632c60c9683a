"""Runs the C2-sized conv kernels (fprop, dgrad, wgrad) a few times, for ncu / timing.

    python tools/prof_conv.py [--n 256] [--c 64] [--iters 5] [--math fp32]
"""
import argparse
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp  # noqa: E402
from paper_2009_01462_b200._lib import lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--hw", type=int, default=32)
ap.add_argument("--c", type=int, default=64)
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--math", default="fp32")
ap.add_argument("--which", default="fprop,dgrad,wgrad")
ap.add_argument("--kernel", type=int, default=-1, help="plane convs: 1 conv_pm, 0 conv_tc, -1 default")
a = ap.parse_args()
lib().rp_op_set_plane_conv_kernel(a.kernel)
n, h, w, c = a.n, a.hw, a.hw, a.c
dev = torch.device("cuda")
x = torch.randn(n, h, w, c, device=dev)
g = torch.randn(n, h, w, c, device=dev)
out = torch.empty_like(x)
wt = torch.randn(3, 3, c, c, device=dev) * 0.05
b = torch.zeros(c, device=dev)
ws_b = max(lib().rp_op_conv3x3_workspace_bytes(c, c), lib().rp_op_conv3x3_wgrad_workspace_bytes(n, h, w, c, c))
ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
gw = torch.empty(3, 3, c, c, device=dev)
gb = torch.empty(c, device=dev)
ne = n * h * w * c
xp = torch.empty(2 * ne, dtype=torch.float16, device=dev)   # plane pairs: p1 = p0 + ne
gp = torch.empty(2 * ne, dtype=torch.float16, device=dev)
planes = [xp[:ne], xp[ne:], gp[:ne], gp[ne:]]
for src, (p0, p1) in ((x, planes[:2]), (g, planes[2:])):
    rp.check(lib().rp_op_split_planes(C.c_void_p(src.data_ptr()), src.numel(), C.c_void_p(p0.data_ptr()),
                                      C.c_void_p(p1.data_ptr()), None, None))
ws_p = lib().rp_op_conv3x3_wgrad_planes_workspace_bytes(n, h, w, c, c)
ws_b = max(ws_b, ws_p, lib().rp_op_conv3x3_wgrad_bf16p_workspace_bytes(n, h, w, c, c))
ws = torch.empty(ws_b, dtype=torch.uint8, device=dev)
P = C.c_void_p
m = rp.MATH[a.math]
flops = 2 * 9 * c * c * n * h * w
for which in a.which.split(","):
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for it in range(a.iters + 1):
        if it == 1:
            torch.cuda.synchronize()
            ev0.record()
        if which == "fprop":
            rp.check(lib().rp_op_conv3x3(n, h, w, c, c, P(x.data_ptr()), P(wt.data_ptr()), 0, P(b.data_ptr()), None,
                                         1.0, 1, P(out.data_ptr()), m, P(ws.data_ptr()), ws_b, None))
        elif which == "dgrad":
            rp.check(lib().rp_op_conv3x3(n, h, w, c, c, P(g.data_ptr()), P(wt.data_ptr()), 1, None, P(x.data_ptr()),
                                         1.0, 3, P(out.data_ptr()), m, P(ws.data_ptr()), ws_b, None))
        elif which in ("fprop_planes", "dgrad_planes"):
            d = which == "dgrad_planes"
            rp.check(lib().rp_op_conv3x3_planes(n, h, w, c, c, P(planes[0].data_ptr()), P(wt.data_ptr()), int(d),
                                                P(b.data_ptr()), P(x.data_ptr()) if d else None, 1.0, 3 if d else 1,
                                                P(out.data_ptr()), P(planes[2].data_ptr()), None, None,
                                                P(ws.data_ptr()), ws_b, None))
        elif which == "wgrad_bf16p":
            rp.check(lib().rp_op_conv3x3_wgrad_bf16p(n, h, w, c, c, C.c_void_p(planes[0].data_ptr()),
                                                     C.c_void_p(planes[2].data_ptr()), 1.0, P(gw.data_ptr()),
                                                     P(gb.data_ptr()), P(ws.data_ptr()), ws_b, None))
        elif which == "wgrad_planes":
            rp.check(lib().rp_op_conv3x3_wgrad_planes(n, h, w, c, c, *[C.c_void_p(t.data_ptr()) for t in planes], 1.0,
                                                      None, P(gw.data_ptr()), P(gb.data_ptr()), P(ws.data_ptr()), ws_b,
                                                      None))
        else:
            rp.check(lib().rp_op_conv3x3_wgrad(n, h, w, c, c, P(x.data_ptr()), P(g.data_ptr()), 1.0,
                                               P(gw.data_ptr()), P(gb.data_ptr()), m, P(ws.data_ptr()), ws_b, None))
    ev1.record()
    torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / a.iters
    print(f"{which}: {ms * 1e3:.1f} us/launch, {flops / ms / 1e9:.1f} TFLOP/s (fp32-equivalent)")
