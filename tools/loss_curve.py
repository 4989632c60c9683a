"""Loss per step of the decoupled trainer on a config's synthetic batch (stability check).

    python tools/loss_curve.py [C2] [steps]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2009_01462_b200 as rp  # noqa: E402
from paper_2009_01462_b200._lib import lib  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 15
cfg = dict(bench.CONFIGS[cfgname])
g = rp.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], bench.CLASSES)
B, K = cfg["B"], cfg["K"]
variants = [("paper", {}), ("kappa_lr=0", {"kappa_lr": 0.0}), ("lambda_lr=0", {"lambda_lr": 0.0}),
            ("lr=0", {"lr": 0.0}), ("penalty", {"mode": rp.PENALTY}), ("kappa_lr=6e-12", {"kappa_lr": 6e-12}),
            ("kappa_lr=1e-10", {"kappa_lr": 1e-10}), ("kappa_lr=1e-12", {"kappa_lr": 1e-12}),
            ("kappa_lr=1e-13", {"kappa_lr": 1e-13}), ("kappa_lr=1e-14", {"kappa_lr": 1e-14})]
if len(sys.argv) > 3:
    variants = [v for v in variants if v[0] in sys.argv[3].split(",")]
for name, over in variants:
    mode = over.pop("mode", rp.ALM)
    tr = rp.DecoupledTrainer(g, K, mode, rp.SQUARED_L2, B, seed_state=bench._splitmix(1), math="fp32")
    x = torch.empty(B * g.raw_size, dtype=torch.float32, device="cuda")
    st = C.c_uint64(1000)
    rp.check(lib().rp_op_fill_uniform(C.c_void_p(x.data_ptr()), x.numel(), C.byref(st), -1.0, 1.0, 1.0, None))
    y = torch.randint(0, 10, (B,), dtype=torch.int32, device="cuda")
    xh = x.cpu().numpy().reshape(B, -1)
    tr.reset_lambda_from_forward(xh.reshape(B, cfg["h"], cfg["w"], cfg["cin"]))
    sp = bench.step_params(cfg)
    for k, v in over.items():
        setattr(sp, k, v)
    losses = [tr.step(xh, y.cpu().numpy(), 0, sp) for _ in range(steps)]
    print(f"{name:14s}", " ".join(f"{v:.3g}" for v in losses))
