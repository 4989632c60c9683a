"""Microbenchmark of conv_tc.cu's fprop MMA pattern in isolation (cycles per MMA)."""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_01462_b200 import _lib
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))  # tools/umma_probe/build.sh
out = torch.zeros(148, device="cuda")
for mode, name in ((89, "collector"), (88, "no collector"), (87, "collector+commit/stage")):
    for lbo in (374,):
        rc = L.rp_debug_umma_bench(2, 128, 0, 0, 2, 3600, 2, mode, lbo, 148, C.c_void_p(out.data_ptr()))
        print(f"fprop pattern {name:24s} halo LBO {lbo:4d} pos: {float(out.mean()):6.1f} cyc/MMA rc={rc}")
