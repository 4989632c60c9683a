"""Serial full backprop (K = 1, serial_train_step) vs layer-parallel (K = 2 / 4 / 8) of the SAME
64-block network (3x32x32, B 256, C 64) on one B200, in one process, with
the same data, step parameters and kernels: timed images/s (CUDA graphs; stages sharing
the GPU on concurrent streams) and per-class kernel times from an untimed profiled pass.

    python tools/serial_vs_parallel.py [--lr 0.005] [--steps 60] [--ks 1,2,4,8]
"""
import argparse, ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib
from paper_2009_01462_b200.trainer import SerialTrainer

ap = argparse.ArgumentParser()
ap.add_argument("--lr", type=float, default=0.002)
ap.add_argument("--steps", type=int, default=60)
ap.add_argument("--ks", default="1,2,4,8")
ap.add_argument("--mode", default="alm")
ap.add_argument("--both", action="store_true", help="K > 1 also with the stages serialised on one stream")
ap.add_argument("--batch", type=int, default=None, help="override C3's B (per-launch fixed-cost study)")
a = ap.parse_args()
cfg = dict(bench.CONFIGS["C3"])
cfg["lr"] = a.lr
if a.batch:
    cfg["B"] = a.batch
B = cfg["B"]
g = rp.Geometry(3, 32, 32, 64, 64, 64, 10)
x, y = bench.synthetic_data(cfg, B, 1000, torch, rp, lib)
xh = x.cpu().numpy().reshape(B, 32, 32, 3)
rows = []
for K in [int(k) for k in a.ks.split(",")]:
    for conc in ((False, True) if (K > 1 and a.both) else ((True,) if K > 1 else (False,))):
        os.environ["RP_CONCURRENT_STAGES"] = "1" if conc else "0"
        if K == 1:
            tr = SerialTrainer(g, B, seed_state=bench._splitmix(1))
            sp = rp.StepParams(beta=1.0, lr=a.lr, lambda_lr=0.0, kappa_lr=0.0)
        else:
            mode = rp.ALM if a.mode == "alm" else rp.PENALTY
            tr = rp.DecoupledTrainer(g, K, mode, rp.SQUARED_L2, B, seed_state=bench._splitmix(1))
            c = dict(cfg)
            c["K"] = K
            sp = bench.step_params(c)
        os.environ.pop("RP_CONCURRENT_STAGES", None)
        tr.reset_lambda_from_forward(xh)
        tr.use_cuda_graphs(True)
        for _ in range(5):
            tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp)
        torch.cuda.synchronize()
        bench.settle(lambda: tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp), 1.0, torch.cuda.synchronize)
        clocks = bench.ClockSampler(0)
        clocks.start()
        rp.check(lib().rp_trainer_region(tr._h, 0, None))
        for _ in range(a.steps):
            tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp)
        ms = C.c_float()
        rp.check(lib().rp_trainer_region(tr._h, 1, C.byref(ms)))
        clk = clocks.stop()
        loss = tr.last_loss()
        # profiled pass (eager, serialised kernels on their own events)
        tr.use_cuda_graphs(False)
        lib().rp_profile_enable(1)
        bench.profile_classes()
        for _ in range(3):
            tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp)
        torch.cuda.synchronize()
        lib().rp_profile_enable(0)
        prof = bench.profile_classes()
        row = {"K": K, "B": B, "concurrent": conc, "img_s": B * a.steps / (ms.value / 1e3), "ms_step": ms.value / a.steps,
               "loss": loss, "lr": a.lr, "sm_mhz": clk["sm_mhz"], "clock_reasons": clk["reasons"],
               "classes_ms": {k: round(v["ms"] / 3, 3) for k, v in prof.items()},
               "conv_tflops": {k: round(v["flops"] / (v["ms"] / 1e3) / 1e12, 1) for k, v in prof.items()
                               if k.startswith("conv_")}}
        print(json.dumps(row), flush=True)
        rows.append(row)
        tr.close()
        del tr
        torch.cuda.empty_cache()
