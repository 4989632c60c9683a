#!/usr/bin/env python
"""Mutation check of the parity tests: build deliberately broken copies of the library and
show that the GPU parity tests FAIL against them (a test suite that still passes on a
broken kernel proves nothing).

    python tools/mutation_check.py build              # here (nvcc cross-compiles), -> tools/_mut/<name>/
    python tools/mutation_check.py run [tests...]     # on the GPU box: every mutant must fail

Each mutant is one textual change in a copy of paper_2009_01462_b200/csrc; the copy is built
with the package's own build.py into tools/_mut/<name>/librespar_b200.so (git-ignored, but it
travels to the GPU box with the snapshot) and the tests load it through RP_LIB_PATH.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "tools", "_mut")
PKG = "paper_2009_01462_b200"

MUTANTS = {
    # the low plane of the scaled cotangent pair (the synthetic / loss upstream the first
    # backward conv and the weight gradients read)
    "cotangent_p1_zero": ("csrc/kernels/conv_wgrad_planes.cu",
                          "    pack_pair4(vv, sc, p0[i], p1[i]);\n  }\n}\n\ntypedef",
                          "    pack_pair4(vv, sc, p0[i], p1[i]);\n    p1[i] = make_uint2(0u, 0u);\n  }\n}\n\ntypedef"),
    # the multiplier term of the synthetic upstream, one lane of four
    "kappa_term_sign": ("csrc/kernels/elementwise.cu",
                        "o.x = -dlam(kind, l.x - xe.x, 0, -1) * w + k4.x;",
                        "o.x = -dlam(kind, l.x - xe.x, 0, -1) * w - k4.x;"),
    # the weight scale divided out of the plane conv epilogue off by 2^-16 (a 1.5e-5 relative bias)
    "epilogue_scale_bias": ("csrc/kernels/conv_pm.cu",
                            "const float acc_mul = kWeightPlaneScaleInv / ",
                            "const float acc_mul = (kWeightPlaneScaleInv * (1.f + 0x1p-16f)) / "),
    # CTA pairs: the peer holds W0 channels [0, 32) instead of [32, 64) for the x1 product (an
    # error at the 2^-11 relative level of the low plane, in half the output channels)
    "pair_x1_half": ("csrc/kernels/conv_pm.cu",
                     "bulk_load(dct + 2048, sct + rank * 512, 512, w_full);",
                     "bulk_load(dct + 2048, sct, 512, w_full);"),
    # the weight-gradient reduce sums the wrong CTAs' partials under the CTA-triple mapping
    "triples_reduce_stride": ("csrc/kernels/conv_wgrad_planes.cu",
                              "first = 3 * c_lo + gi, stride = 3, count = c_hi - c_lo;",
                              "first = 3 * c_lo + gi, stride = 1, count = c_hi - c_lo;"),
    # the 16-channel weight gradient accumulates its first K-step onto stale TMEM
    "wsmall_stale_accumulator": ("csrc/kernels/conv_wgrad_small.cu",
                                 "tap == kBiasTap ? id_b : id, (first && k == 0) ? 0u : 1u);",
                                 "tap == kBiasTap ? id_b : id, 1u);"),
    # the per-thread plane stores (the Co = 64 default) swap the two 16-byte halves of every
    # 32-byte low-plane sector (channels 8 apart trade their low planes)
    "direct_plane_halves": ("csrc/kernels/conv_pm.cu",
                            "stg256(a.p1 + off + hf * kCh + 16 * j, cat2(h1[0], h1[1]), cat2(h1[2], h1[3]));",
                            "stg256(a.p1 + off + hf * kCh + 16 * j, cat2(h1[2], h1[3]), cat2(h1[0], h1[1]));"),
}

DEFAULT_TESTS = ["tests/test_gpu_plane_parity.py", "tests/test_gpu_block_planes.py",
                 "tests/test_gpu_configs.py::test_config_three_iterations"]


def build():
    for name, (rel, old, new) in MUTANTS.items():
        d = os.path.join(OUT, name)
        shutil.rmtree(d, ignore_errors=True)
        shutil.copytree(os.path.join(ROOT, PKG), os.path.join(d, PKG),
                        ignore=shutil.ignore_patterns("_build", "*.so", "__pycache__"))
        shutil.copytree(os.path.join(ROOT, "include"), os.path.join(d, "include"))
        src = os.path.join(d, PKG, rel)
        text = open(src).read()
        if text.count(old) != 1:
            raise SystemExit(f"{name}: pattern not found exactly once in {rel}")
        open(src, "w").write(text.replace(old, new))
        r = subprocess.run([sys.executable, os.path.join(d, PKG, "build.py")], capture_output=True, text=True)
        if r.returncode != 0:
            raise SystemExit(f"{name}: build failed\n{r.stderr[-3000:]}")
        lib = os.path.join(d, PKG, "librespar_b200.so")
        shutil.move(lib, os.path.join(d, "librespar_b200.so"))
        shutil.rmtree(os.path.join(d, PKG))
        shutil.rmtree(os.path.join(d, "include"))
        print(f"built {name}")


def run(tests):
    ok = True
    for name in MUTANTS:
        lib = os.path.join(OUT, name, "librespar_b200.so")
        env = {**os.environ, "RP_LIB_PATH": lib}
        r = subprocess.run([sys.executable, "-m", "pytest", "-q", "-m", "gpu", "-p", "no:cacheprovider", *tests],
                           env=env, capture_output=True, text=True, cwd=ROOT)
        tail = [ln for ln in r.stdout.splitlines() if "passed" in ln or "failed" in ln][-1:]
        # caught = the tests ran and failed (not an import or collection error)
        caught = r.returncode == 1 and bool(tail) and "failed" in tail[0]
        ok &= caught
        print(f"{name}: {'CAUGHT' if caught else 'NOT CAUGHT'} ({tail[0] if tail else r.stdout[-300:]})")
    return ok


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "build":
        build()
    else:
        sys.exit(0 if run(sys.argv[2:] or DEFAULT_TESTS) else 1)
