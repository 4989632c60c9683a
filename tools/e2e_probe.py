"""Why can the e2e loop (host buffers, a synchronising loss read per step) beat the device-timed
graph-replay loop?  C3 trainer, 100 steps each way, wall clock + SM clock samples:
  a) step_device back to back (graph replay, no per-step sync) -- bench's timed region
  b) step_device + loss read each step (per-step sync)
  c) step with host arrays (H2D staging + loss read) -- bench's e2e
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib

cfg = dict(bench.CONFIGS["C3"])
B, K = cfg["B"], cfg["K"]
g = rp.Geometry(3, 32, 32, 64, 64, 64, 10)
os.environ["RP_CONCURRENT_STAGES"] = "1"
tr = rp.DecoupledTrainer(g, K, rp.ALM, rp.SQUARED_L2, B, seed_state=bench._splitmix(1))
os.environ.pop("RP_CONCURRENT_STAGES")
x, y = bench.synthetic_data(cfg, B, 1000, torch, rp, lib)
xh = x.cpu().numpy().reshape(B, -1)
yh = y.cpu().numpy()
tr.reset_lambda_from_forward(xh)
sp = bench.step_params(cfg)
tr.use_cuda_graphs(True)
for _ in range(5):
    tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp)
torch.cuda.synchronize()
bench.settle(lambda: tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp), 2.0, torch.cuda.synchronize)
for rep in range(2):
    for mode in ("a", "b", "c", "a"):
        clk = bench.ClockSampler(0)
        clk.start()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(100):
            if mode == "a":
                tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp)
            elif mode == "b":
                tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=True)
            else:
                tr.step(xh, yh, 0, sp)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        c = clk.stop()
        print(f"{mode}: {B * 100 / dt:8.0f} img/s  {dt * 10:.2f} ms/step  sm {c['sm_mhz']} MHz", flush=True)
