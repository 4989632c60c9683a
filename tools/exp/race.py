import hashlib, sys, os
import numpy as np
import torch
sys.path.insert(0, "/root/repo")
import paper_2009_01462_b200 as rp
from oracle import respar_oracle as O
graphs = os.environ.get("GRAPHS", "1") == "1"
g = rp.Geometry(3, 16, 16, 64, 64, 8, 10)
x, y = O.synthetic_batch(O.Geometry(3, 16, 16, 64, 64, 8, 10), 32, 3)
xs = np.ascontiguousarray(x, np.float32)
tr = rp.DecoupledTrainer(g, 4, rp.ALM, rp.SQUARED_L2, 32, seed_state=11)
tr.reset_lambda_from_forward(xs)
tr.use_cuda_graphs(graphs)
xd = torch.from_numpy(xs).cuda()
yd = torch.from_numpy(y.astype(np.int32)).cuda()
sp = rp.StepParams(beta=0.1, lr=0.05, lambda_lr=0.05, kappa_lr=1e-6)
for _ in range(5):
    tr.step_device(xd.data_ptr(), yd.data_ptr(), 32, 0, sp)
h = hashlib.sha256(tr.params().tobytes() + b"".join(tr.state(k, rp.LAMBDA).tobytes() for k in range(1, 4)))
print(os.environ.get("RP_CONCURRENT_STAGES", "0"), os.environ.get("RP_PDL", "1"), graphs, h.hexdigest()[:16], tr.last_loss())
