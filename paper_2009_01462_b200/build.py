"""Builds the in-tree shared library paper_2009_01462_b200/librespar_b200.so.

nvcc -gencode arch=compute_100a,code=sm_100a (sm_100a only: the tcgen05/TMA kernels
do not exist on any other target), -lineinfo for ncu source mapping.  Objects are
compiled in parallel and cached by content hash under paper_2009_01462_b200/_build/.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "librespar_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-I" + os.path.join(ROOT, "include"),
          "-I" + CSRC, "--expt-relaxed-constexpr", "-Xcompiler", "-Wall,-Wno-unused-function"]


def sources():
    out = []
    for d, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cu", ".cpp")):
                out.append(os.path.join(d, f))
    return sorted(out)


def headers():
    hs = [os.path.join(ROOT, "include", "respar_b200.h")]
    for d, _, files in os.walk(CSRC):
        hs += [os.path.join(d, f) for f in files if f.endswith((".h", ".hpp", ".cuh"))]
    return sorted(hs)


def _digest(path, extra):
    h = hashlib.sha256()
    with open(path, "rb") as f:
        h.update(f.read())
    h.update(extra)
    return h.hexdigest()[:16]


def _compile(src, hdr_digest, verbose):
    rel = os.path.relpath(src, CSRC).replace(os.sep, "_")
    flags = ARCH + COMMON + (["-Xptxas", "-v"] if os.environ.get("RP_PTXAS_V") else [])
    key = _digest(src, hdr_digest + " ".join(flags).encode())
    obj = os.path.join(BUILD, f"{rel}.{key}.o")
    if os.path.exists(obj):
        return obj, None
    cmd = [NVCC] + flags + ["-c", src, "-o", obj + ".tmp"]
    if src.endswith(".cpp"):
        cmd = [NVCC] + flags + ["-x", "c++", "-c", src, "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj, (r.stderr if verbose else None)


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    if force:
        shutil.rmtree(BUILD)
        os.makedirs(BUILD)
    hd = hashlib.sha256()
    for h in headers():
        with open(h, "rb") as f:
            hd.update(f.read())
    hdr_digest = hd.digest()
    srcs = sources()
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        results = list(ex.map(lambda s: _compile(s, hdr_digest, verbose), srcs))
    objs = [o for o, _ in results]
    for _, log in results:
        if log:
            sys.stderr.write(log)
    link_key = hashlib.sha256("".join(objs).encode()).hexdigest()[:16]
    stamp = os.path.join(BUILD, "link.stamp")
    if os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == link_key:
        return LIB
    cmd = [NVCC] + ARCH + ["-shared", "-o", LIB + ".tmp"] + objs + ["-lcuda", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(LIB + ".tmp", LIB)
    with open(stamp, "w") as f:
        f.write(link_key)
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="--force" in sys.argv))
