"""Loss per step through the bench's own setup (device-resident synthetic batch, step_device).

    python tools/loss_steps.py [C5] [steps]
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2009_01462_b200 as rp  # noqa: E402
from paper_2009_01462_b200._lib import lib  # noqa: E402

cfgname = sys.argv[1] if len(sys.argv) > 1 else "C5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 12
cfg = dict(bench.CONFIGS[cfgname])
g = rp.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], bench.CLASSES)
B, K = cfg["B"], cfg["K"]
if cfg["mode"] == "serial":
    from paper_2009_01462_b200.trainer import SerialTrainer
    tr = SerialTrainer(g, B, seed_state=bench._splitmix(1), math=cfg["math"])
else:
    mode = {"alm": rp.ALM, "penalty": rp.PENALTY}[cfg["mode"]]
    tr = rp.DecoupledTrainer(g, K, mode, rp.SQUARED_L2, B, seed_state=bench._splitmix(1), math=cfg["math"])
x = torch.empty(B * g.raw_size, dtype=torch.float32, device="cuda")
st = C.c_uint64(1000)
rp.check(lib().rp_op_fill_uniform(C.c_void_p(x.data_ptr()), x.numel(), C.byref(st), -1.0, 1.0, 1.0, None))
y = torch.randint(0, 10, (B,), dtype=torch.int32, device="cuda")
tr.reset_lambda_from_forward(x.cpu().numpy().reshape(B, cfg["h"], cfg["w"], cfg["cin"]))
sp = bench.step_params(cfg)
if os.environ.get("LR"):
    sp.lr = float(os.environ["LR"])
tr.use_cuda_graphs(os.environ.get("GRAPHS", "0") == "1")
losses = [tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=True) for _ in range(steps)]
print(cfgname, "lr", sp.lr, os.environ.get("RP_BF16_TAPE", "tape"), "graphs" if os.environ.get("GRAPHS") == "1" else "eager", " ".join(f"{v:.4g}" for v in losses))
