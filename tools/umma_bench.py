"""tcgen05.mma tf32 issue-rate microbenchmark (cycles per MMA, 148 CTAs, one per SM).

    python tools/umma_bench.py
"""
import ctypes as C, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2009_01462_b200 import _lib
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))  # tools/umma_probe/build.sh
out = torch.zeros(148, device="cuda")
cases = []
for N in (32, 64, 128, 256):
    for taps in (3,):
        for mode, what in ((92, "no collector"), (90, "A collector fill/use/lastuse")):
            cases.append((f"wgrad N={N} taps={taps} {what}", 2, N, 3, 1, 2, taps, mode, 1))
for name, fmt, N, layout, amn, bmn, nacc, mode, chain in cases:
    if nacc * N > 512:
        continue
    rc = L.rp_debug_umma_bench(fmt, N, layout, amn, bmn, 3600, nacc, mode, chain, 148, C.c_void_p(out.data_ptr()))
    cyc = float(out.mean())
    print(f"tf32 {name:50s} rc={rc}: {cyc:6.1f} cyc/MMA (ideal {N / 2:5.1f}) -> {128*N*8/cyc:5.0f} MAC/clk/SM")
