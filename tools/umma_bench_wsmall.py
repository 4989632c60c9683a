"""MMA rate of the 16-channel wgrad pattern (conv_wgrad_small.cu): M64/M128 x N x K16, MN-major
no-swizzle operands, 9 shifted taps per K-step into 9 column blocks (148 CTAs).

    bash tools/umma_probe/build.sh && python tools/umma_bench_wsmall.py
"""
import ctypes as C, os
import torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))
out = torch.zeros(148, device="cuda")
def run(nops, N, layout, chain=232):
    rc = L.rp_debug_umma_bench(0, N, layout, 1, 1, 9 * 400, 2, nops, chain, 148, C.c_void_p(out.data_ptr()))
    assert rc == 0, rc
    return float(out.mean())
for N in (32, 40, 48):
    print(f"N={N}: M64 mn {run(60, N, 4):6.1f}  M128 mn {run(60, N, 0):6.1f}  M64 one-block {run(61, N, 4):6.1f}  "
          f"M64 kmajor {run(62, N, 4):6.1f}  M64 no-shift {run(63, N, 4):6.1f} cyc/MMA")
