"""Cycles per tcgen05.mma (kind::f16, M = 128, K = 16, 148 CTAs) as a function of N: is the
MMA time linear in N or quantised (the conv's equal 224-position units vs 256 + a tail)?

    bash tools/umma_probe/build.sh && python tools/umma_bench_n.py
"""
import ctypes as C, os, sys
import torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))
out = torch.zeros(148, device="cuda")
for fmt, name in ((0, "f16"), (1, "bf16")):
    for N in (16, 32, 48, 64, 96, 128, 160, 176, 192, 208, 224, 240, 256):
        rc = L.rp_debug_umma_bench(fmt, N, 0, 0, 0, 4096, 2, 86, 1, 148, C.c_void_p(out.data_ptr()))
        cyc = float(out.mean())
        print(f"{name} N={N:3d}: {cyc:6.1f} cyc/MMA (linear {N / 2:5.1f}) rc={rc}", flush=True)
