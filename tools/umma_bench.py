import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_01462_b200 import _lib
L = C.CDLL(_lib.LIB_PATH)
out = torch.zeros(148, device="cuda")
for N in (128, 256):
    for mode, name in ((97, "A same, no collector"), (98, "A collector fill/use/lastuse")):
        rc = L.rp_debug_umma_bench(2, N, 0, 0, 0, 4000, 2, mode, 1, 148, C.c_void_p(out.data_ptr()))
        cyc = float(out.mean())
        print(f"tf32 N={N} {name} rc={rc}: {cyc:6.1f} cyc/MMA -> {128*N*8/cyc:5.0f} MAC/clk/SM")
