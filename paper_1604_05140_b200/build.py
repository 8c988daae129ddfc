"""In-tree build of the sm_100a library (libsglb200.so) and its C++ test driver.

    python -m paper_1604_05140_b200.build

nvcc cross-compiles for sm_100a without a GPU; the .so is written next to this
file so it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libsglb200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CUDA_SOURCES = ["sgl_kernels.cu", "sgl_separated.cu", "sgl_ozaki.cu", "sgl_small.cu"]
CXX_SOURCES = ["sgl_tables.cpp", "sgl_capi.cpp", "sgl_api.cpp", "sgl_host.cpp"]


def _sources():
    return [os.path.join(CSRC, s) for s in CUDA_SOURCES + CXX_SOURCES]


def _headers():
    hs = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".hpp", ".h"))]
    inc = os.path.join(REPO, "include")
    for root, _d, files in os.walk(inc):
        hs += [os.path.join(root, f) for f in files]
    return hs


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    deps = _sources() + _headers() + [os.path.abspath(__file__)]
    target = out or LIB
    if not force and not _stale(target, deps):
        return target
    # variant builds (--out=) get their own object directory so they can run in parallel
    objdir = os.path.join(PKG, "_obj", os.path.basename(out)) if out else os.path.join(PKG, "_obj")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    common = ["-O3", "-std=c++20", "-Xcompiler", "-fPIC,-pthread", "-I", os.path.join(REPO, "include"),
              "-I", CSRC] + [f for f in os.environ.get("SGL_NVCC_FLAGS", "").split() if f]
    procs = []
    for src in _sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        objs.append(obj)
        cmd = [NVCC] + ARCH + common + ["-lineinfo", "-c", src, "-o", obj]
        if src.endswith(".cpp"):
            cmd = [NVCC] + common + ["-x", "c++", "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out.decode())
            raise RuntimeError("build failed: " + " ".join(cmd))
    tmp = target + ".tmp"
    link = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-lcudart", "-Xcompiler", "-pthread"]
    subprocess.run(link, check=True)
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    outs = [a.split("=", 1)[1] for a in sys.argv[1:] if a.startswith("--out=")]
    print(build(force="--force" in sys.argv, verbose=True, out=outs[0] if outs else None))
