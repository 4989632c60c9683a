"""Per step: loss, max |param| / |grad|, and max |.| of every stage state (lambda, kappa,
boundary_out, boundary_adjoint) -- where a non-finite value first appears.

    python tools/nan_hunt.py [C5] [steps]
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2009_01462_b200 as rp  # noqa: E402
from paper_2009_01462_b200._lib import lib  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 22
cfg = dict(bench.CONFIGS[cfgname])
g = rp.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], bench.CLASSES)
B, K = cfg["B"], cfg["K"]
tr = rp.DecoupledTrainer(g, K, rp.ALM, rp.SQUARED_L2, B, seed_state=bench._splitmix(1), math=cfg["math"])
x = torch.empty(B * g.raw_size, dtype=torch.float32, device="cuda")
st = C.c_uint64(1000)
rp.check(lib().rp_op_fill_uniform(C.c_void_p(x.data_ptr()), x.numel(), C.byref(st), -1.0, 1.0, 1.0, None))
gen = torch.Generator(device="cuda")
gen.manual_seed(7)
y = torch.randint(0, 10, (B,), dtype=torch.int32, device="cuda", generator=gen)
tr.reset_lambda_from_forward(x.cpu().numpy().reshape(B, cfg["h"], cfg["w"], cfg["cin"]))
sp = bench.step_params(cfg)


C_, Ch_, Cin_ = cfg["c"], cfg["ch"], cfg["cin"]
S_W = 9 * Cin_ * C_
BLK0 = S_W + C_
BSTR = 9 * C_ * Ch_ + Ch_ + 9 * Ch_ * C_ + C_


def where(i):
    if i < S_W:
        return "stem.w"
    if i < BLK0:
        return "stem.b"
    if i < BLK0 + BSTR * cfg["L"]:
        l, r = divmod(i - BLK0, BSTR)
        part = "w1" if r < 9 * C_ * Ch_ else "b1" if r < 9 * C_ * Ch_ + Ch_ else "w2" if r < 9 * C_ * Ch_ + Ch_ + 9 * Ch_ * C_ else "b2"
        return f"block{l}.{part}"
    return "head"


def mx(a):
    a = np.asarray(a, dtype=np.float64)
    if a.size == 0:
        return "-"
    return "nan" if not np.all(np.isfinite(a)) else f"{np.abs(a).max():.3g}"


for i in range(steps):
    loss = tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=True)
    p, gr = tr.params(), tr.grads()
    ag = np.abs(np.nan_to_num(gr.astype(np.float64), nan=np.inf))
    parts = [f"step {i:2d} loss {loss:.5g} |p| {mx(p)} |g| {mx(gr)} at {where(int(ag.argmax()))}"]
    for k in range(K if os.environ.get("STATES") else 0):
        s = [mx(tr.state(k, w)) for w in range(4)]
        parts.append(f"k{k}:" + "/".join(s))
    print(" ".join(parts), flush=True)
    if not np.isfinite(loss):
        break
