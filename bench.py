#!/usr/bin/env python
"""Benchmark: train images/sec of one layer-parallel training iteration
(DecoupledTrainer::step, reference decoupled.cpp:172-194) on B200.

Default: BASELINE.json configs[2] == SURVEY §8 C3, the metric's own network: ODE-ResNet
3x32x32, batch 256, C = 64, L = 64 residual blocks, K = 8 stages, augmented Lagrangian
(kappa updates), fp32 math, full batch (N_train = B).  At N = 1 the 8 stages share the GPU
(concurrent streams); at N = 2/4/8 stage k runs on GPU floor(k N / 8) with the neighbour
exchange over NCCL (N = 8: one stage per B200).  Inputs are synthetic (the reference's
splitmix64 stream: pixels U[-1,1), then labels next_u64() % 10) and device-resident for
`value`; `e2e` times the same step through the public C ABI with pinned host buffers (H2D of
x and labels, D2H of the loss inside the timed region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config C3]

--gpus N without a torchrun environment re-launches itself under torch.distributed.run
with N ranks (one per GPU); under torchrun, WORLD_SIZE must equal N.

`--impl reference` times the reference's own CPU trainer (oracle/_ref, compiled from
the reference sources) on the same config's dense 1x1-conv analogue, a bounded sample
of images per step.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # id: (Cin, H, W, C, Ch, L, K, B, mode, math, classes)
    "C1": dict(cin=1, h=28, w=28, c=16, ch=16, L=8, K=2, B=128, mode="penalty", math="fp32"),
    # lr 0.1 fits C2's repeated batch through loss spikes (0.002 .. 7 at the end of a run, by step
    # count); 0.01 keeps it smooth
    "C2": dict(cin=3, h=32, w=32, c=64, ch=64, L=16, K=4, B=256, mode="alm", math="fp32", concurrent=True, lr=0.01),
    # the 64-block network on one repeated synthetic batch: at lr 0.1 the layer-parallel step
    # diverges after ~170 steps (C3) and serial backprop within ~15 (C4); at 0.005 the serial one
    # after ~500.  lr 0.002 keeps both finite for > 1,000 steps (tools/clock_timeline.py, loss per
    # window) -- a benchmark on non-finite data is void: the tensor pipe draws less power on NaN
    # and the capped clock jumps from ~1.5 to ~1.9 GHz (profiles/r02_clock_timeline.txt)
    "C3": dict(cin=3, h=32, w=32, c=64, ch=64, L=64, K=8, B=256, mode="alm", math="fp32", concurrent=True, lr=0.002),
    "C4": dict(cin=3, h=32, w=32, c=64, ch=64, L=64, K=1, B=256, mode="serial", math="fp32", lr=0.002),
    "C5": dict(cin=3, h=32, w=32, c=256, ch=256, L=64, K=8, B=1024, mode="alm", math="bf16"),
}
CLASSES = 10
METRIC = "train images/sec at K=1/2/4/8 B200 stages; conv tensor-pipe % of peak"


def flops_per_image(cfg):
    """108 C^2 HW per block (6 conv-equivalents) + stem fprop/wgrad."""
    hw = cfg["h"] * cfg["w"]
    return cfg["L"] * 6 * 2 * 9 * cfg["c"] * cfg["ch"] * hw + 2 * 2 * 9 * cfg["cin"] * cfg["c"] * hw


# effective multiplier step kappa_lr * # / (2 beta) of the bench's ALM runs (see step_params)
KAPPA_STEP = 1e-8


def step_params(cfg):
    import paper_2009_01462_b200 as rp
    # paper schedules at epoch 0 (config.cpp:102-111): ALM beta 0.1, penalty beta 1; lr 0.1;
    # lambda_lr = lr * lambda_lr_scale (1.0).  kappa_lr: the multiplier step is
    # kappa_lr * # / (2 beta) with # = rows x features (decoupled.cpp:157-170).  The reference's
    # 1e-9 is sized for its 2-D toy (# = 200 x 8: a step of 8e-6); on a conv stage # = B H W C
    # (16.8 M at C2) makes the same kappa_lr a 1e4 x larger step and the iteration diverges to
    # inf / nan within ~8 steps (tools/loss_curve.py) -- timing a benchmark on non-finite data
    # is meaningless (the tensor pipe draws less power on it).  The bench therefore keeps the
    # effective step at KAPPA_STEP, which stays finite over the whole bench run (every kernel
    # of the ALM step still runs; the value only sets the multiplier's step size).
    beta = 0.1 if cfg["mode"] == "alm" else 1.0
    n = cfg["B"] * cfg["h"] * cfg["w"] * cfg["c"]
    kappa_lr = KAPPA_STEP * 2.0 * beta / n
    lr = cfg.get("lr", 0.1)
    return rp.StepParams(beta=beta, tau=-1.0, lr=lr, lambda_lr=lr, kappa_lr=kappa_lr, max_corrections=1)


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.isfile(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def profile_classes():
    from paper_2009_01462_b200._lib import lib
    n = 9
    launches = (C.c_int64 * n)()
    ms = (C.c_double * n)()
    fl = (C.c_double * n)()
    by = (C.c_double * n)()
    from paper_2009_01462_b200 import check
    check(lib().rp_profile_collect(launches, ms, fl, by))
    out = {}
    for i in range(n):
        if launches[i]:
            out[lib().rp_profile_class_name(i).decode()] = dict(launches=launches[i], ms=ms[i], flops=fl[i],
                                                              bytes=by[i])
    return out


def run_ours(args, cfg, rank, world):
    import numpy as np
    import torch

    import paper_2009_01462_b200 as rp
    from paper_2009_01462_b200._lib import lib

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    g = rp.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], CLASSES)
    B, K = cfg["B"], cfg["K"]
    mode = {"alm": rp.ALM, "penalty": rp.PENALTY, "serial": rp.SERIAL}[cfg["mode"]]
    # train(): root = Rng(seed); net_rng = root.split() (decoupled.cpp:274-276), seed 1
    from paper_2009_01462_b200.trainer import SerialTrainer
    net_state = _splitmix(1)
    # Stages sharing a GPU run on concurrent streams for the timed run where that is faster
    # (cfg "concurrent": the small C = 64 convs leave SMs idle in every kernel's tail, which a
    # neighbouring stage's kernels fill); the roofline pass below uses a serialised trainer so
    # every kernel's event-timed duration is its own.
    concurrent = (bool(cfg.get("concurrent")) or args.concurrent_stages) and not args.serial_stages

    def make_trainer(conc):
        os.environ["RP_CONCURRENT_STAGES"] = "1" if conc else "0"
        try:
            if mode == rp.SERIAL:
                return SerialTrainer(g, B, seed_state=net_state, math=args.math or cfg["math"])
            return rp.DecoupledTrainer(g, K, mode, rp.SQUARED_L2, B, seed_state=net_state,
                                       math=args.math or cfg["math"])
        finally:
            os.environ.pop("RP_CONCURRENT_STAGES", None)

    tr = make_trainer(concurrent)
    # synthetic data, device-resident, from the reference's RNG stream (seed 1000 + replica)
    x, y = synthetic_data(cfg, B, 1000 + rank, torch, rp, lib)
    x_host = x.cpu().numpy().reshape(B, cfg['h'], cfg['w'], cfg['cin'])
    tr.reset_lambda_from_forward(x_host)
    sp = step_params(cfg)
    tr.use_cuda_graphs(not args.no_graphs)   # the step is captured once and replayed

    for _ in range(args.warmup):
        tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=False)
    torch.cuda.synchronize()
    settle_steps, settle_s, settle_mhz = settle(
        lambda: tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=False), args.settle_s,
        torch.cuda.synchronize, dev)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()

    # timed region: no per-kernel event records inside it
    clocks = ClockSampler(dev)
    clocks.start()
    n0 = rp.launch_count()
    h = tr._h
    rp.check(lib().rp_trainer_region(h, 0, None))
    for _ in range(args.steps):
        tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=False)
    ms = C.c_float()
    rp.check(lib().rp_trainer_region(h, 1, C.byref(ms)))
    torch.cuda.synchronize()
    launches = rp.launch_count() - n0
    clk = clocks.stop()
    total_ms = ms.value
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    loss = tr.last_loss()

    # e2e through the public API with pinned host buffers (H2D x, labels; D2H loss)
    xp = torch.from_numpy(x_host).pin_memory()
    yp = y.cpu().pin_memory()
    xpn = xp.numpy()
    ypn = yp.numpy()
    e2e_steps = max(1, args.steps)   # as many steps as the timed region: both sustained
    tr.step(xpn.reshape(B, -1), ypn, 0, sp)  # warm the staging buffers
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    loss_e2e = float("nan")
    for _ in range(e2e_steps):
        loss_e2e = tr.step(xpn.reshape(B, -1), ypn, 0, sp)
    torch.cuda.synchronize()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    loss = loss if math.isfinite(loss_e2e) else loss_e2e   # a non-finite e2e loss voids the line too

    # a second, profiled pass of the same step: per-kernel-class CUDA-event times for the
    # roofline (event records on the launching streams; not part of the timed value), on a
    # serialised trainer
    if concurrent:
        tr.close()
        del tr
        import gc
        gc.collect()
        tr = make_trainer(False)
        tr.reset_lambda_from_forward(x_host)
    tr.use_cuda_graphs(False)                # per-kernel events need eager launches
    lib().rp_profile_enable(1)
    profile_classes()  # clear
    prof_steps = min(args.steps, 5)
    for _ in range(prof_steps):
        tr.step_device(x.data_ptr(), y.data_ptr(), B, 0, sp, read_loss=False)
    torch.cuda.synchronize()
    lib().rp_profile_enable(0)
    prof = profile_classes()
    return dict(tr=tr, total_ms=total_ms, prof=prof, clocks=clk, launches=launches, loss=loss, e2e_s=e2e_s,
                B=B, K=K, g=g, prof_steps=prof_steps, concurrent=concurrent, settle=(settle_steps, settle_s, settle_mhz))


def run_ours_distributed(args, cfg, rank, world):
    """N > 1: one process per GPU, stage k of the K-stage pipeline on rank floor(k G / K)
    (paper_2009_01462_b200/distributed.py: placement); N > K runs N / K pipeline replicas, each
    on its own synthetic batch.  The step runs on the C++-host NCCL pipeline
    (NcclStagePipeline, csrc/host/pipeline.hpp): chunked p / lambda transfers on dedicated
    streams overlapped with the corrections, the whole step replayed from one CUDA graph."""
    import torch
    import torch.distributed as dist
    import paper_2009_01462_b200 as rp
    from paper_2009_01462_b200._lib import lib
    from paper_2009_01462_b200.distributed import NcclStagePipeline, placement

    dev = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(dev)
    g = rp.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], CLASSES)
    B, K = cfg["B"], cfg["K"]
    if cfg["mode"] == "serial":
        raise SystemExit("bench: the serial config runs on one GPU (K = 1)")
    mode = {"alm": rp.ALM, "penalty": rp.PENALTY}[cfg["mode"]]
    plc = placement(K, world, rank)
    # several stages per rank (N < K): concurrent stage streams as at N = 1
    concurrent = ((bool(cfg.get("concurrent")) or args.concurrent_stages) and not args.serial_stages
                  and plc.hi - plc.lo > 1)
    os.environ["RP_CONCURRENT_STAGES"] = "1" if concurrent else "0"
    try:
        tr = NcclStagePipeline.for_rank(g, K, mode, rp.SQUARED_L2, B, plc, dev, seed_state=_splitmix(1),
                                        math=args.math or cfg["math"], chunks=args.chunks)
    finally:
        os.environ.pop("RP_CONCURRENT_STAGES", None)
    x, y = synthetic_data(cfg, B, 1000 + plc.replica, torch, rp, lib)
    tr.reset_lambda_from_forward(x.data_ptr() if plc.first else None)
    sp = step_params(cfg)
    tr.set_graphs(not args.no_graphs)
    xp = x.data_ptr() if plc.first else None
    yp = y.data_ptr() if plc.last else None
    for _ in range(args.warmup):
        tr.step(xp, yp, B, 0, sp)
    tr.sync()
    settle_steps, settle_s, settle_mhz = settle(lambda: tr.step(xp, yp, B, 0, sp), args.settle_s, tr.sync, dev)
    dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(dev)
    clocks.start()
    n0 = rp.launch_count()
    tr.region(0)
    for _ in range(args.steps):
        tr.step(xp, yp, B, 0, sp)
    total_ms = tr.region(1)
    launches = rp.launch_count() - n0
    clk = clocks.stop()
    t = torch.tensor([total_ms], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    # the last stage's loss, to every rank (a scalar, off the data path)
    lt = torch.tensor([tr.loss() if plc.last else 0.0], dtype=torch.float64, device="cuda")
    dist.all_reduce(lt, op=dist.ReduceOp.SUM)
    loss = float(lt.item()) / max(1, plc.replicas)

    # e2e: pinned host batch -> device (stage-0 rank: pixels, last-stage rank: labels), the
    # step, the loss read back on the last-stage rank; wall clock, max over ranks
    x_host = x.cpu().pin_memory()
    y_host = y.cpu().pin_memory()
    e2e_steps = max(1, args.steps)   # as many steps as the timed region: both sustained
    dist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        if plc.first:
            x.copy_(x_host, non_blocking=True)
        if plc.last:
            y.copy_(y_host, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        tr.step(xp, yp, B, 0, sp, read_loss=True)
    tr.sync()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], device="cuda")
    dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)

    # profiled pass for the roofline classes (untimed, eager launches)
    tr.set_graphs(False)
    lib().rp_profile_enable(1)
    profile_classes()
    prof_steps = min(args.steps, 5)
    for _ in range(prof_steps):
        tr.step(xp, yp, B, 0, sp)
    tr.sync()
    lib().rp_profile_enable(0)
    prof = profile_classes()
    return dict(tr=tr, total_ms=total_ms, prof=prof, clocks=clk, launches=launches, loss=loss,
                e2e_s=float(e2e_s.item()), B=B, K=K, g=g, replicas=plc.replicas, plc=plc, prof_steps=prof_steps,
                concurrent=concurrent, prof_concurrent=concurrent, settle=(settle_steps, settle_s, settle_mhz))


def reference_labels(seed, n_before, count):
    """next_u64() % 10 for draws n_before .. n_before + count - 1 of Rng(seed)
    (tensor.cpp:163-169: draw i = mix(seed + (i + 1) gamma))."""
    M = (1 << 64) - 1
    out = []
    for j in range(count):
        z = (seed + (n_before + j + 1) * 0x9E3779B97F4A7C15) & M
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        out.append((z ^ (z >> 31)) % CLASSES)
    return out


def synthetic_data(cfg, B, seed, torch, rp, lib):
    """The reference's synthetic batch (acceptance.cpp:69-73 pattern): pixels
    rng_uniform(B H W Cin, -1, 1) from Rng(seed) (tensor.cpp:177-185; filled on device by the
    same splitmix64 stream), then labels next_u64() % 10 from the draws that follow."""
    n = B * cfg["h"] * cfg["w"] * cfg["cin"]
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    st = C.c_uint64(seed)
    rp.check(lib().rp_op_fill_uniform(C.c_void_p(x.data_ptr()), n, C.byref(st), -1.0, 1.0, 1.0, None))
    y = torch.tensor(reference_labels(seed, n, B), dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    return x, y


def settle(step_fn, seconds, sync, gpu=0, max_seconds=20.0):
    """Untimed steps beyond the warm-up until the SM clock has settled: at least `seconds`, then
    until three consecutive ~0.5 s windows agree on the median SM clock within 1.5 % (nvidia-smi,
    100 ms samples), at most `max_seconds`.  Returns (steps, seconds, [window medians])."""
    sampler = ClockSampler(gpu)
    sampler.start()
    n = 0
    t0 = time.perf_counter()
    meds = []
    while True:
        w0 = time.perf_counter()
        mark = len(sampler.lines)
        while time.perf_counter() - w0 < 0.5:
            step_fn()
            n += 1
            if n % 4 == 0:
                sync()
        sync()
        el = time.perf_counter() - t0
        win = [ln for ln in sampler.lines[mark:]]
        clk = []
        for ln in win:
            try:
                clk.append(float(ln.split(",")[0]))
            except (ValueError, IndexError):
                pass
        if clk:
            meds.append(sorted(clk)[len(clk) // 2])
        if seconds <= 0 or el >= max_seconds or (el >= seconds and sampler.proc is None):
            break
        if el >= seconds and len(meds) >= 3 and max(meds[-3:]) - min(meds[-3:]) <= 0.015 * max(meds[-3:]):
            break
    sampler.stop()
    return n, time.perf_counter() - t0, meds


def _splitmix(seed):
    """Rng(seed).split().state == Rng(seed).next_u64() (tensor.cpp:163-175)."""
    M = (1 << 64) - 1
    z = (seed + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def cpu_reference_sample(cfg, images, workers):
    """The reference's own DecoupledTrainer::step (oracle/_ref) on the dense 1x1-conv
    analogue of cfg (rows = images*H*W, d = C, h = Ch, same L, K, mode): seconds/step."""
    from oracle import refbind as R
    hw = cfg["h"] * cfg["w"]
    rows = images * hw
    dims = (cfg["cin"], cfg["c"], cfg["ch"], cfg["L"], CLASSES)
    rng = R.RefRng(1)
    params = R.make_net(rng, *dims)
    x = rng.uniform(rows, cfg["cin"], -1.0, 1.0)
    import numpy as np
    y = np.array([rng.next_u64() % CLASSES for _ in range(rows)], np.int32)
    mode = {"alm": 2, "penalty": 1, "serial": 1}[cfg["mode"]]
    K = cfg["K"]
    tr = R.RefTrainer(dims, 0, params, K, mode, 0, rows, workers=workers)
    tr.reset_lambda_from_forward(x)
    beta = 0.1 if cfg["mode"] == "alm" else 1.0
    t0 = time.perf_counter()
    kappa_lr = KAPPA_STEP * 2.0 * beta / (rows * cfg["c"])   # the same multiplier step as step_params
    tr.step(x, y, 0, beta=beta, tau=-1.0, lr=0.1, lambda_lr=0.1, kappa_lr=kappa_lr, max_corrections=1)
    return time.perf_counter() - t0


def cpu_port_sample(cfg, images):
    """The CPU restatement of the same 3x3-conv step (oracle/respar_oracle.py, numpy fp64, the
    checker the parity tests use) on a sample of `images`: seconds per step.  Secondary CPU
    baseline: the reference itself has no convolution."""
    import numpy as np
    from oracle import respar_oracle as O
    og = O.Geometry(cfg["cin"], cfg["h"], cfg["w"], cfg["c"], cfg["ch"], cfg["L"], CLASSES)
    net = O.make_net(og, O.Rng(1))
    x, y = O.synthetic_batch(og, images, seed=1000)
    mode = {"alm": O.ALM, "penalty": O.PENALTY, "serial": O.PENALTY}[cfg["mode"]]
    tr = O.DecoupledTrainer(net, cfg["K"], mode, O.SQUARED_L2, images)
    tr.reset_lambda_from_forward(x)
    beta = 0.1 if cfg["mode"] == "alm" else 1.0
    t0 = time.perf_counter()
    tr.step(x, y, 0, O.StepParams(beta=beta, tau=-1.0, lr=cfg.get("lr", 0.1), lambda_lr=cfg.get("lr", 0.1),
                                  kappa_lr=KAPPA_STEP * 2.0 * beta / (images * og.feature_size)))
    return time.perf_counter() - t0


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    from oracle import refbind as R
    if not R.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/librespar_ref.so not built"}))
        return
    workers = min(cfg["K"], os.cpu_count() or 1)
    images = max(1, args.ref_images)
    times = []
    for i in range(args.warmup + args.steps):
        t = cpu_reference_sample(cfg, images, workers)
        if i >= args.warmup:
            times.append(t)
    per_step = statistics.mean(times)
    v = images / per_step
    line = {
        "metric": METRIC, "value": v, "unit": "images/s", "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config}: reference DecoupledTrainer::step (fp64 CPU) on the dense 1x1-conv "
                               f"analogue rows=images*H*W", **_cfg_json(cfg),
                   "sample_images_per_step": images,
                   "ms_per_step_is": f"the measured time of one step on the {images}-image sample"},
        "cpu_baseline": {"value": v, "unit": "images/s", "cores": workers, "kind": "reference",
                         "sample": f"{images} image(s) x {cfg['h']}x{cfg['w']} rows per step, one "
                                   f"DecoupledTrainer::step, StagePool with {workers} workers"},
        "e2e": {"value": v, "unit": "images/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def _cfg_json(cfg):
    beta = 0.1 if cfg["mode"] == "alm" else 1.0
    n = cfg["B"] * cfg["h"] * cfg["w"] * cfg["c"]
    operands = {"fp32": "fp16x2 plane pairs (22-bit significands, power-of-two scales), fp32 accumulate; "
                        "fprop / dgrad 3 tensor products per MAC (positions-as-M conv_pm.cu, C <= 64; "
                        "x0 W0 + x0 W1 + x1 W0), wgrad 4 ([g0; g1] x [x0 x1])",
                "bf16": "bf16 operands, fp32 accumulate", "tf32": "tf32 operands, fp32 accumulate",
                "simt": "fp32 CUDA cores"}[cfg["math"]]
    return {"in": [cfg["cin"], cfg["h"], cfg["w"]], "global_batch": cfg["B"], "channels": cfg["c"],
            "hidden": cfg["ch"], "blocks": cfg["L"], "stages": cfg["K"], "mode": cfg["mode"],
            "math": cfg["math"], "conv_operands": operands, "classes": CLASSES, "lr": cfg.get("lr", 0.1),
            "beta": beta, "lambda_lr": cfg.get("lr", 0.1),
            "kappa_lr": KAPPA_STEP * 2.0 * beta / n if cfg["mode"] == "alm" else None,
            "kappa_step": KAPPA_STEP if cfg["mode"] == "alm" else None, "penalty": "squared_l2",
            "data_rng": "reference splitmix64 (seed 1000 + replica): pixels U[-1,1), then labels next_u64() % 10"}


def plane_conv_products(cfg):
    """Tensor products per fp32 MAC of the config's plane convs: 3 on conv_pm.cu, 4 on conv_tc.cu."""
    from paper_2009_01462_b200._lib import lib
    kinds = {lib().rp_op_plane_conv_kernel(cfg["B"], cfg["h"], cfg["w"], ci, co)
             for ci, co in ((cfg["c"], cfg["ch"]), (cfg["ch"], cfg["c"]))}
    return 3 if kinds == {1} else 4


def spawn_ranks(n, check_devices=True):
    """--gpus N outside torchrun: re-launch this command under torch.distributed.run with N
    ranks (one per GPU, rendezvous on 127.0.0.1); the ranks' output is this process's."""
    import socket
    try:
        import torch
        avail = torch.cuda.device_count()
    except Exception:
        avail = 0
    if check_devices and avail < n:
        raise SystemExit(f"bench: --gpus {n} but only {avail} CUDA device(s) are visible")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.run(cmd).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C3", choices=sorted(CONFIGS))
    ap.add_argument("--settle-s", type=float, default=1.5,
                    help="untimed steps after the warm-up for at least this many seconds, then until the SM clock "
                         "is steady; 0 disables")
    ap.add_argument("--chunks", type=int, default=4, help="N > 1: row chunks of the p / lambda exchange")
    ap.add_argument("--cpu-port-images", type=int, default=1,
                    help="images of the 3x3 CPU restatement sample (secondary CPU baseline; 0 disables)")
    ap.add_argument("--math", default=None, choices=[None, "fp32", "tf32", "bf16", "simt"])
    ap.add_argument("--ref-images", type=int, default=2)
    ap.add_argument("--cpu-images", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graphs", action="store_true", help="launch every kernel eagerly (no CUDA graph replay)")
    ap.add_argument("--concurrent-stages", action="store_true",
                    help="stages sharing a GPU on streams of their own even where the config does not")
    ap.add_argument("--serial-stages", action="store_true",
                    help="stages sharing the GPU on one stream also in the timed run (default: concurrent for C2/C3)")
    ap.add_argument("--plan", action="store_true",
                    help="print each rank's stages and neighbours (one JSON line per rank) and exit: the launcher "
                         "and placement without a GPU")
    ap.add_argument("--dist-path", action="store_true",
                    help="run the one-process-per-GPU stage-sharded path even at N=1 (smoke of the N>1 code)")
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.math:
        cfg["math"] = args.math
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))

    if args.impl == "reference":
        # the reference arm is a CPU run: rank 0 alone (the other ranks of a torchrun exit 0)
        run_reference(args, cfg, rank, world)
        return

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus, check_devices=not args.plan))
    if world != args.gpus:
        raise SystemExit(f"bench: --gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or drop the torchrun environment")
    if args.plan:
        from paper_2009_01462_b200.distributed import placement
        plc = placement(cfg["K"], world, rank)
        # one write per line: the ranks share the parent's stdout (print writes text and newline apart)
        sys.stdout.write(json.dumps({"rank": rank, "world": world, "local_rank": int(os.environ.get("LOCAL_RANK", "0")),
                                     "stages": [plc.lo, plc.hi], "prev_rank": plc.prev_rank,
                                     "next_rank": plc.next_rank, "replica": plc.replica,
                                     "replicas": plc.replicas}) + "\n")
        sys.stdout.flush()
        return

    distributed = world > 1 or args.dist_path
    if distributed:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29517")
            dist.init_process_group("nccl", rank=rank, world_size=world)

    r = run_ours_distributed(args, cfg, rank, world) if distributed else run_ours(args, cfg, rank, world)
    if rank != 0:
        return
    B, K = r["B"], r["K"]
    replicas = r.get("replicas", 1)
    total_s = r["total_ms"] / 1e3
    value = replicas * B * args.steps / total_s   # every pipeline replica ran B images per step
    peaks, peaks_kind = measured_peaks()
    prof = r["prof"]
    convs = {k: v for k, v in prof.items() if k.startswith("conv_")}
    dom = max(convs, key=lambda k: convs[k]["ms"]) if convs else max(prof, key=lambda k: prof[k]["ms"])
    d = prof[dom]
    avg_ms = d["ms"] / d["launches"]
    achieved_tf = d["flops"] / d["launches"] / (avg_ms / 1e3) / 1e12
    ps = r["prof_steps"]
    step_prof_ms = sum(v["ms"] for v in prof.values()) / ps
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.isfile(tpath):
        with open(tpath) as f:
            tj = json.load(f)
            t = tj.get(f"{args.config}:{dom}") or tj.get(dom)
        traffic = t["bytes_per_launch"] if t else None
    # the fp32-accurate kernels run every fp32 MAC as 4 fp16 tensor products (the plane path:
    # [W0; W1] x {x0, x1} in fprop / dgrad, [g0; g1] x [x0 x1] in wgrad; fp16
    # and bf16 MMAs run at the same rate): their own ceiling is the 16-bit peak / 4, reported
    # beside the prescribed bf16-peak fraction together with the tensor work actually issued
    split = {"fp32": 4.0, "tf32": 2.0, "bf16": 1.0, "simt": None}.get(cfg["math"])
    if cfg["math"] == "fp32" and dom != "conv_wgrad" and plane_conv_products(cfg) == 3:
        split = 3.0   # the positions-as-M plane conv drops the W1 x1 product
    ceiling = peaks["bf16_tflops_sustained"] / split if split else None
    roof = {"bound": "tensor", "kernel": dom, "achieved": achieved_tf,
            "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
            "frac": achieved_tf / peaks["bf16_tflops_sustained"], "traffic": traffic,
            "traffic_unit": "bytes per launch (ncu --set full, profiles/traffic.json)",
            "math_ceiling": {"tflops": ceiling, "frac": achieved_tf / ceiling if ceiling else None,
                             "tensor_tflops_issued": achieved_tf * split if split else None,
                             "products_per_mac": split,
                             "note": "bf16 sustained peak / 16-bit tensor products per fp32-equivalent MAC "
                                     "(fp32 plane path: fprop / dgrad 3 (conv_pm) or 4 (conv_tc), wgrad 4; bf16: 1)"},
            "peak_source": f"{peaks_kind} bf16 dense sustained (MEASURED_PEAKS.json)",
            "kernel_timing": ("per-launch CUDA events with this rank's stages on concurrent streams (overlapping "
                              "kernels: upper bounds)") if r.get("prof_concurrent") else
                             "per-launch CUDA events, stages serialised (untimed pass)",
            "avg_launch_ms": avg_ms, "launches": d["launches"],
            "share_of_step": d["ms"] / ps / step_prof_ms if step_prof_ms else None,
            "kernel_classes": {k: {"launches": v["launches"], "ms_per_step": v["ms"] / ps,
                                   "tflops": (v["flops"] / (v["ms"] / 1e3) / 1e12) if v["ms"] and v["flops"] else None,
                                   "gbs": (v["bytes"] / (v["ms"] / 1e3) / 1e9) if v["ms"] and v["bytes"] else None}
                               for k, v in prof.items()}}
    flops_iter = flops_per_image(cfg) * B
    line = {
        "metric": METRIC, "value": value, "unit": "images/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": r["total_ms"] / args.steps, "higher_is_better": True,
        # N <= K: one pipeline, the same batch spread over more GPUs; N > K: replicas
        "scaling": "weak" if world > K else "strong", "vs_baseline": None,
        "dtype": "bf16" if cfg["math"] == "bf16" else "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: ODE-ResNet {cfg['cin']}x{cfg['h']}x{cfg['w']}, batch {B}, "
                               f"C={cfg['c']}, L={cfg['L']}, K={K} stages, {cfg['mode']}, math {cfg['math']}",
                   **_cfg_json(cfg),
                   "parallelism": f"{K} stages on {min(world, K)} GPU(s) (stage k on rank floor(k G / K); N > 1: "
                                  f"C++-host NCCL point-to-point exchange of p / lambda in {args.chunks} chunks on "
                                  f"dedicated streams, CUDA-graph replay)" + (f" x {replicas} replicas" if replicas > 1
                                                                             else "")
                                  + ("; stages sharing a GPU on concurrent streams" if r.get("concurrent") else ""),
                   "l2": "inputs larger than L2 (per-iteration working set > 2 GB)",
                   "model_flops_per_iter": flops_iter,
                   "model_tflops": flops_iter * replicas * args.steps / total_s / 1e12},
        # the reference's ALM update (kappa_lr 1e-9, lambda_lr 0.1) diverges on this synthetic
        # batch after ~10 iterations - the reference itself does the same (tools/ref_loss_curve.py);
        # a non-finite value is reported as null so the line stays valid JSON
        "loss": r["loss"] if math.isfinite(r["loss"]) else None,
        # the timed and e2e steps must run on finite data (a diverged step draws different power)
        "diverged": not math.isfinite(r["loss"]),
        "clocks": r["clocks"],
        "gpu_launches": r["launches"],
        "roofline": roof,
        "e2e": {"value": replicas * B / r["e2e_s"], "unit": "images/s",
                "h2d_bytes_per_step": replicas * (B * r["g"].raw_size * 4 + B * 4),
                "d2h_bytes_per_step": 8 * replicas, "steps": args.steps,
                "timing": "wall clock around the steps, each step: H2D of pixels and labels from pinned "
                          "host memory, the step, D2H of the loss (synchronising)"},
    }
    line["config"]["settle"] = {"untimed_steps": r["settle"][0], "seconds": round(r["settle"][1], 3),
                                "sm_mhz_windows": r["settle"][2][-12:],
                                "note": "after the W warm-up steps, before the K timed steps: at least --settle-s, "
                                        "then until three ~0.5 s windows agree on the median SM clock within 1.5 %"}
    if not args.no_cpu_baseline and args.cpu_port_images > 0:
        try:
            t = cpu_port_sample(cfg, args.cpu_port_images)
            line["cpu_baseline_3x3"] = {"value": args.cpu_port_images / t, "unit": "images/s", "cores": os.cpu_count(),
                                        "kind": "port",
                                        "sample": f"{args.cpu_port_images} image(s) of the 3x3-conv network, one step "
                                                  f"of oracle/respar_oracle.py (numpy fp64, BLAS threads)"}
        except Exception as e:  # reported, never fatal
            line["cpu_baseline_3x3"] = {"value": None, "unit": "images/s", "sample": f"failed: {e}"}
    if not args.no_cpu_baseline:
        try:
            workers = min(K, os.cpu_count() or 1)
            t = cpu_reference_sample(cfg, args.cpu_images, workers)
            line["cpu_baseline"] = {"value": args.cpu_images / t, "unit": "images/s", "cores": workers,
                                    "kind": "reference",
                                    "sample": f"{args.cpu_images} images (rows = images*{cfg['h']}*{cfg['w']}) "
                                              f"of the dense 1x1-conv analogue, one reference "
                                              f"DecoupledTrainer::step (fp64), {workers} StagePool workers"}
        except Exception as e:  # reported, never fatal
            line["cpu_baseline"] = {"value": None, "unit": "images/s", "cores": 0, "kind": "reference",
                                    "sample": f"failed: {e}"}
    if line.get("diverged"):
        print("bench: the loss went non-finite during the timed / e2e steps -- the line is void (lower the "
              "config's lr)", file=sys.stderr)
    print(json.dumps(line))


def _shutdown():
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()
    except Exception:
        pass


if __name__ == "__main__":
    try:
        main()
    finally:
        _shutdown()
