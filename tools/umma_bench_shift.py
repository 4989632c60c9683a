import ctypes as C, os, sys
import torch
sys.path.insert(0, "/root/repo")
from paper_2009_01462_b200 import _lib
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))  # tools/umma_probe/build.sh
out = torch.zeros(148, device="cuda")
for chain in (1, 2, 4, 8, 256):
    for bmn in (0, 2):
        rc = L.rp_debug_umma_bench(2, 128, 0, 0, bmn, 3600, 2, 96, chain, 148, C.c_void_p(out.data_ptr()))
        print(f"K-major interleave N=128 A same, B shifts of {chain} x16B, data {'rand' if bmn == 2 else 'const'}: {float(out.mean()):6.1f} cyc/MMA rc={rc}")
