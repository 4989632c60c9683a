"""bf16 tcgen05.mma rate for the conv_tc PLANES issue pattern (M=128, N=256, K=16; A = weight
tap through the collector, B = shifted halo plane views), 148 CTAs.  Ideal: 128 cycles/MMA.

    python tools/umma_bench_planes.py
"""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_01462_b200 import _lib
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))  # tools/umma_probe/build.sh
out = torch.zeros(148, device="cuda")
for nops, what in ((80, "shifted B, collector"), (81, "aligned B, collector"), (82, "shifted B, no collector")):
    for bmn, data in ((0, "const"), (2, "random")):
        rc = L.rp_debug_umma_bench(1, 256, 0, 0, bmn, 6000, 2, nops, 374, 148, C.c_void_p(out.data_ptr()))
        print(f"planes pattern {what:26s} data {data:6s}: {float(out.mean()):6.1f} cyc/MMA (ideal 128) rc={rc}")
