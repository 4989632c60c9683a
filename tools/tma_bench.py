"""TMA load throughput by box shape (148 CTAs, one box in flight per ring slot): the conv halo's
16-byte rows ({8 ch, W + 1, rows, C / 8 groups}) against 32 / 64 / 128-byte rows.

    bash tools/umma_probe/build.sh && python tools/tma_bench.py
"""
import ctypes as C, os
import torch
L = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "umma_probe", "librp_probe.so"))
out = torch.zeros(148, device="cuda")
n, h, w, c = 256, 32, 32, 64
x = torch.randn(n, h, w, c, device="cuda").half()
iters = 200
for depth in (2, 4, 6):
    for cg, rows in ((8, 11), (8, 22), (16, 11), (16, 22), (32, 11), (64, 5)):
        rc = L.rp_debug_tma_bench(C.c_void_p(x.data_ptr()), n, h, w, c, cg, rows, iters, depth, C.c_void_p(out.data_ptr()))
        assert rc == 0, rc
        cyc = float(out.max())
        ngroups = 2 if cg == 8 else 1
        rowb = 16 if cg == 8 else 2 * cg
        nrows = (w + 1) * rows * ngroups
        box = rowb * nrows
        print(f"depth {depth} rows of {rowb:3d} B x {nrows:5d} = {box:6d} B/box: {cyc / iters:7.1f} cyc/box, "
              f"{box * iters / cyc:6.1f} B/cyc/SM, {cyc / iters / nrows:5.2f} cyc/row", flush=True)
