import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
from oracle import refbind as R
import bench
cfg = bench.CONFIGS["C2"]
for images, steps in ((16, 30), (64, 15)):
    rows = images * 1024
    dims = (cfg["cin"], cfg["c"], cfg["ch"], cfg["L"], 10)
    rng = R.RefRng(1)
    params = R.make_net(rng, *dims)
    x = rng.uniform(rows, cfg["cin"], -1.0, 1.0)
    y = np.array([rng.next_u64() % 10 for _ in range(rows)], np.int32)
    tr = R.RefTrainer(dims, 0, params, 4, 2, 0, rows, workers=4)
    tr.reset_lambda_from_forward(x)
    out = []
    t0 = time.time()
    for s in range(steps):
        out.append(tr.step(x, y, 0, beta=0.1, tau=-1.0, lr=0.1, lambda_lr=0.1, kappa_lr=1e-9, max_corrections=1))
    print(images, "images", f"{time.time()-t0:.1f}s", " ".join(f"{v:.3g}" for v in out), flush=True)
