"""After reset_lambda_from_forward, stage 0's synthetic upstream is exactly 0 at the first
step, so every stage-0 gradient must be 0.  Prints the max |grad| of stage 0's range."""
import ctypes as C, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib

B, L, K, c, hw = (int(v) for v in sys.argv[1:6])
g = rp.Geometry(3, hw, hw, c, c, L, 10)
tr = rp.DecoupledTrainer(g, K, rp.ALM, rp.SQUARED_L2, B, seed_state=bench._splitmix(1), math="bf16")
x = torch.empty(B * g.raw_size, dtype=torch.float32, device="cuda")
st = C.c_uint64(1000)
rp.check(lib().rp_op_fill_uniform(C.c_void_p(x.data_ptr()), x.numel(), C.byref(st), -1.0, 1.0, 1.0, None))
y = torch.randint(0, 10, (B,), dtype=torch.int32, device="cuda")
tr.reset_lambda_from_forward(x.cpu().numpy().reshape(B, hw, hw, 3))
out0 = tr.state(0, rp.BOUNDARY_OUT).copy()
sp = bench.step_params(dict(bench.CONFIGS["C5"], B=B, h=hw, w=hw, c=c))
tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=True)
grads = tr.grads()
blk0 = 9 * 3 * c + c
bstride = 2 * (9 * c * c + c)
n0 = blk0 + (L // K) * bstride
out1 = tr.state(0, rp.BOUNDARY_OUT)
print(f"B={B} L={L} K={K} C={c} hw={hw} tape={os.environ.get('RP_BF16_TAPE', '1')}: stage-0 max|grad| "
      f"{np.abs(grads[:n0]).max():.3e} (stem {np.abs(grads[:blk0]).max():.3e}); X0_end step vs reset max diff "
      f"{np.abs(out1 - out0).max():.3e}")
