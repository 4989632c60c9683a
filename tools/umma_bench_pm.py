"""MMA time of the positions-as-M plane conv pattern (conv_pm) against the channels-as-M one
(conv_tc PLANES): cycles per tap and 256 positions, 148 CTAs.

    bash tools/umma_probe/build.sh && python tools/umma_bench_pm.py
"""
import ctypes as C, os
import torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))
out = torch.zeros(148, device="cuda")
def run(nops, N, reps, chain=300):
    rc = L.rp_debug_umma_bench(0, N, 0, 0, 0, reps, 2, nops, chain, 148, C.c_void_p(out.data_ptr()))
    assert rc == 0, rc
    return float(out.mean())
for _ in range(2):
    c80 = run(80, 256, 6 * 600)
    print(f"channels-as-M (conv_tc PLANES, 2 x N=256 per tap): {2 * c80:7.1f} cyc per tap / 256 positions")
    c82 = run(82, 256, 6 * 600)
    print(f"  same without the A collector:                  {2 * c82:7.1f}")
    for co in (64, 32, 16):
        N = 2 * co
        c70 = run(70, N, 12 * 300)
        c71 = run(71, N, 12 * 300)
        c72 = run(72, N, 6 * 300)
        print(f"positions-as-M Co={co}: x0 N={N} + x1 N={co}: {4 * c70:7.1f}   both N={N}: {4 * c71:7.1f}   "
              f"x0 only: {2 * c72:7.1f} cyc per tap / 256 positions")
