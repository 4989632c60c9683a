"""GPU: examples/cpp_drop_in.cpp -- a compiled C++ caller of the C++ mirror of the reference API
 -- builds against librespar_b200.so, runs, and its losses equal the Python
front end's on the same seeds bit for bit; the reference's exception types come through."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

import paper_2009_01462_b200 as rp
from paper_2009_01462_b200._lib import lib

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_drop_in_example(tmp_path):
    pkg = os.path.join(ROOT, "paper_2009_01462_b200")
    exe = str(tmp_path / "cpp_drop_in")
    cmd = ["/usr/local/cuda/bin/nvcc", "-std=c++17", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(pkg, "csrc"), os.path.join(ROOT, "examples", "cpp_drop_in.cpp"), "-L", pkg, "-lrespar_b200",
           f"-Xlinker=-rpath={pkg}", "-o", exe]
    b = subprocess.run(cmd, capture_output=True, text=True)
    assert b.returncode == 0, b.stderr[-3000:]
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-3000:]
    out = r.stdout.splitlines()
    losses = [float(ln.split()[2]) for ln in out if ln.startswith("loss ")]
    assert "invalid_argument ok" in out and "ConfigError ok" in out
    assert any(ln.startswith("stage0 grads begin 0 size ") for ln in out)
    # the same run through the Python front end
    g = rp.Geometry(3, 8, 8, 64, 64, 4, 10)
    tr = rp.DecoupledTrainer(g, 2, rp.ALM, rp.SQUARED_L2, 8, seed_state=12345)
    x = torch.empty(8 * 8 * 8 * 3, device="cuda")
    st = C.c_uint64(777)
    rp.check(lib().rp_op_fill_uniform(C.c_void_p(x.data_ptr()), x.numel(), C.byref(st), -1.0, 1.0, 1.0, None))
    y = torch.tensor([i % 10 for i in range(8)], dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    tr.reset_lambda_from_forward(x.cpu().numpy().reshape(8, 8, 8, 3))
    sp = rp.StepParams(beta=0.5, lr=0.05, lambda_lr=0.05, kappa_lr=1e-6)
    want = [tr.step_device(x.data_ptr(), y.data_ptr(), 8, 0, sp, read_loss=True) for _ in range(3)]
    assert losses == want, (losses, want)
    assert np.all(np.isfinite(losses))
