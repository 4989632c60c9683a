"""Where an M = 64 tcgen05.mma (kind::f16, cta_group::1) puts D's rows in TMEM (lane of row i)."""
import ctypes as C, os
import numpy as np, torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))
out = torch.zeros(128 * 16, device="cuda")
rc = L.rp_debug_umma_m64_layout(C.c_void_p(out.data_ptr()))
o = out.cpu().numpy().reshape(128, 16)
print("rc", rc)
for lane in range(128):
    print(lane, o[lane, :4])
