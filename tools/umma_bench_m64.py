"""tf32 MMA rate at M = 64 vs M = 128 (K-major interleave, A same, B rotating)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_01462_b200 import _lib
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))  # tools/umma_probe/build.sh
out = torch.zeros(148, device="cuda")
for layout, M in ((0, 128), (4, 64)):
    for N in (128, 256):
        rc = L.rp_debug_umma_bench(2, N, layout, 0, 0, 3600, 2, 97, 1, 148, C.c_void_p(out.data_ptr()))
        cyc = float(out.mean())
        print(f"tf32 M={M} N={N}: {cyc:6.1f} cyc/MMA -> {M * N * 8 / cyc:6.0f} MAC/clk/SM rc={rc}")
