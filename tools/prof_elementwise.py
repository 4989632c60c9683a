"""The HBM-bound kernels of the C3 step at their bench sizes (256 x 32 x 32 x 64 boundary
tensors, one stage's 8 blocks of parameters, the head on 256 images), each launched a few
times -- for ncu's dram__bytes and time (profiles/r02_elementwise.md) and CUDA-event GB/s.

    python tools/prof_elementwise.py [--iters 20]
"""
import argparse, ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=20)
a = ap.parse_args()
P = C.c_void_p
n = 256 * 32 * 32 * 64
dev = torch.device("cuda")
lam, x, kap, p = (torch.rand(n, device=dev) for _ in range(4))
g = torch.empty(n, device=dev)
planes = torch.empty(2 * n, dtype=torch.float16, device=dev)
scale = torch.zeros(lib().rp_op_plane_scale_bytes() // 4, device=dev)
red = torch.empty(lib().rp_op_reduce_workspace_bytes(), dtype=torch.uint8, device=dev)
geo = rp.Geometry(3, 32, 32, 64, 64, 64, 10)
npar = rp.param_count(geo)
stage_params = 8 * (int(lib().rp_param_offset_block(C.byref(geo.c()), 1)) - int(lib().rp_param_offset_block(C.byref(geo.c()), 0)))
w = torch.rand(stage_params, device=dev)
gw = torch.rand(stage_params, device=dev) * 1e-3
B = 256
feat = torch.rand(n, device=dev)
pt = torch.rand(64 * 10 + 10, device=dev) * 0.1
pooled = torch.empty(B * 64, device=dev)
logits = torch.empty(B * 10, device=dev)
labels = torch.randint(0, 10, (B,), dtype=torch.int32, device=dev)
loss = torch.zeros(1, dtype=torch.float64, device=dev)
gt = torch.empty(64 * 10 + 10, device=dev)
wsb = lib().rp_op_workspace_bytes(C.byref(geo.c()), B, 0)
ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
ops = {
    # name: (callable, algorithmic bytes per launch)
    "synthetic_grad_planes (ALM, + scaled fp16 pair)": (lambda: rp.check(lib().rp_op_synthetic_grad_planes(
        0, P(lam.data_ptr()), P(x.data_ptr()), P(kap.data_ptr()), n, 1e-7, P(g.data_ptr()), P(planes.data_ptr()),
        P(planes.data_ptr() + 2 * n), P(scale.data_ptr()), P(red.data_ptr()), None)), 16 * n + 4 * n + 4 * n),
    "correct (lambda + kappa, ALM)": (lambda: rp.check(lib().rp_op_correct(
        0, P(lam.data_ptr()), P(x.data_ptr()), P(p.data_ptr()), P(kap.data_ptr()), n, 1e-7, 0.1, 1, 1e-9, 1,
        P(red.data_ptr()), None)), 24 * n),
    "sgd (one C3 stage, 8 blocks)": (lambda: rp.check(lib().rp_op_sgd(P(w.data_ptr()), P(gw.data_ptr()), None,
                                                                       stage_params, 1e-6, 0.0, None)), 12 * stage_params),
    "head fwd + loss/bwd (GAP, FC, CE, cotangent + scaled pair)": (lambda: (
        rp.check(lib().rp_op_head_fwd(C.byref(geo.c()), B, P(feat.data_ptr()), P(pt.data_ptr()), P(pooled.data_ptr()),
                                      P(logits.data_ptr()), None)),
        rp.check(lib().rp_op_head_loss_bwd_planes(C.byref(geo.c()), B, P(pooled.data_ptr()), P(logits.data_ptr()),
                                                  P(pt.data_ptr()), P(labels.data_ptr()), P(loss.data_ptr()),
                                                  P(gt.data_ptr()), P(g.data_ptr()), P(planes.data_ptr()),
                                                  P(planes.data_ptr() + 2 * n), P(scale.data_ptr()), P(ws.data_ptr()),
                                                  wsb, None))), 4 * n + 4 * n + 4 * n + 4 * n),
}
for name, (fn, by) in ops.items():
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.iters
    print(f"{name}: {ms * 1e3:.1f} us, {by / 1e6:.1f} MB algorithmic, {by / ms / 1e6:.0f} GB/s")
