"""Sustained behaviour of the C3 step: run it back to back (graph replay) for --seconds and print,
per ~2 s window, images/s, the median SM clock, power draw and throttle reasons (nvidia-smi)."""
import argparse, os, subprocess, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib

ap = argparse.ArgumentParser()
ap.add_argument("--seconds", type=float, default=60.0)
ap.add_argument("--config", default="C3")
ap.add_argument("--lr", type=float, default=None, help="override the config's lr")
a = ap.parse_args()
cfg = dict(bench.CONFIGS[a.config])
if a.lr is not None:
    cfg["lr"] = a.lr
B, K = cfg["B"], cfg["K"]
g = rp.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], 10)
os.environ["RP_CONCURRENT_STAGES"] = "1"
mode = {"alm": rp.ALM, "penalty": rp.PENALTY, "serial": rp.SERIAL}[cfg["mode"]]
tr = rp.DecoupledTrainer(g, K, mode, rp.SQUARED_L2, B, seed_state=bench._splitmix(1), math=cfg["math"])
os.environ.pop("RP_CONCURRENT_STAGES")
x, y = bench.synthetic_data(cfg, B, 1000, torch, rp, lib)
tr.reset_lambda_from_forward(x.cpu().numpy().reshape(B, -1))
sp = bench.step_params(cfg)
tr.use_cuda_graphs(True)
for _ in range(3):
    tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp)
torch.cuda.synchronize()
lines = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=timestamp,clocks.sm,power.draw,temperature.gpu,"
                         "clocks_event_reasons.sw_power_cap,clocks_event_reasons.sw_thermal_slowdown,"
                         "clocks_event_reasons.hw_slowdown", "--format=csv,noheader,nounits", "-lms", "200"],
                        stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
threading.Thread(target=lambda: [lines.append((time.time(), l.strip())) for l in proc.stdout], daemon=True).start()
t_start = time.time()
while time.time() - t_start < a.seconds:
    t0 = time.time()
    n = 0
    while time.time() - t0 < 2.0:
        for _ in range(10):
            tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp)
        torch.cuda.synchronize()
        n += 10
    t1 = time.time()
    win = [l for (ts, l) in lines if t0 <= ts <= t1]
    sm = sorted(float(l.split(",")[1]) for l in win if len(l.split(",")) >= 7) or [0.0]
    pw = sorted(float(l.split(",")[2]) for l in win if len(l.split(",")) >= 7) or [0.0]
    tmp = [l.split(",")[3].strip() for l in win if len(l.split(",")) >= 7]
    cap = sum(1 for l in win if len(l.split(",")) >= 7 and "Active" in l.split(",")[4])
    loss = tr.last_loss()
    print(f"t={t0 - t_start:5.1f}s loss {loss:.4g} {B * n / (t1 - t0):8.0f} img/s  sm {sm[len(sm) // 2]:.0f} MHz  "
          f"power {pw[len(pw) // 2]:.0f} W  temp {tmp[-1] if tmp else '?'} C  power-cap samples {cap}/{len(win)}",
          flush=True)
proc.terminate()
