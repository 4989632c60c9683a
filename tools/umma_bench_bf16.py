"""bf16 tcgen05.mma rate on fixed smem operands (148 CTAs): K-major layouts (0 interleave,
6 SW32, 2 SW128), N, and A-operand reuse through the collector.  Ideal M=128 rate: N/2
cycles per MMA.

    python tools/umma_bench_bf16.py
"""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_01462_b200 import _lib
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))  # tools/umma_probe/build.sh
out = torch.zeros(148, device="cuda")
for layout in (0, 2):
    for N in (64, 128, 256):
        for nops, what in ((1, "A re-read"), (85, "4 MMAs same A, no collector"), (86, "4 MMAs same A, collector")):
            rc = L.rp_debug_umma_bench(1, N, layout, 0, 0, 4096, 2, nops, 1, 148, C.c_void_p(out.data_ptr()))
            cyc = float(out.mean())
            print(f"bf16 layout={layout} N={N:3d} {what:30s}: {cyc:6.1f} cyc/MMA (ideal {N / 2:5.1f}) rc={rc}")
