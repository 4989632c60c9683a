import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_gpu_configs import _setup, _oracle
from tests.helpers import rel_err
import paper_2009_01462_b200 as rp
from oracle import respar_oracle as O
cfg, og, p32, x32, y, sp, osp, g = _setup("C2")
K, B = cfg["K"], cfg["B"]
gt = rp.DecoupledTrainer(g, K, rp.ALM, rp.SQUARED_L2, B, params=p32)
gt.reset_lambda_from_forward(x32)
ot, xt = _oracle(og, p32, x32, cfg, K)
yt = torch.from_numpy(y.astype(np.int64)).cuda()
for step in range(3):
    lg = gt.step(x32, y, 0, sp); lo = ot.step(xt, yt, 0, osp)
    print("step", step, "loss", lg, lo, abs(lg-lo)/lo)
    for k in range(K):
        ga = gt.state(k, rp.BOUNDARY_ADJOINT); oa = ot.badj[k].cpu().numpy()
        print(f"  k={k} badj max|want| {np.abs(oa).max():.3e} err {rel_err(ga, oa):.2e}  bout err {rel_err(gt.state(k, rp.BOUNDARY_OUT), ot.bout[k].cpu().numpy()):.2e}")
        if k > 0:
            print(f"       lam err {rel_err(gt.state(k, rp.LAMBDA), ot.lam[k].cpu().numpy()):.2e} kappa max {np.abs(ot.kappa[k].cpu().numpy()).max():.2e} err {rel_err(gt.state(k, rp.KAPPA), ot.kappa[k].cpu().numpy()):.2e}")
