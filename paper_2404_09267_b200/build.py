"""Builds the in-tree CUDA library ``lib/libtangram_gpu.so`` for sm_100a.

Plain nvcc, no Python extension machinery: the library exports the C ABI in
include/tangram_gpu.h and is loaded with ctypes (Python) or linked directly
(C++ drop-in, tests/cpp).  Run ``python -m paper_2404_09267_b200.build``.
"""
from __future__ import annotations

import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBDIR = os.path.join(PKG, "lib")
LIB = os.path.join(LIBDIR, "libtangram_gpu.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [
        os.path.join(ROOT, "include", "tangram_gpu.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Compiles every csrc/*.cu for sm_100a and links lib/libtangram_gpu.so.
    `defines`/`out` build tuning variants (e.g. -DTG_GATHER_PLAN_CHUNKS=4)
    into another file, loaded with TANGRAM_GPU_LIB=<path>."""
    target = out or LIB
    if not force and not defines and out is None and not needs_build():
        return LIB
    os.makedirs(os.path.dirname(target), exist_ok=True)
    objdir = os.path.join(PKG, "_obj" if not defines else "_obj_variant")
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
               "-I", os.path.join(ROOT, "include"), "-I", CSRC, *defines, "-c", src, "-o", obj]
        if verbose:
            cmd[1:1] = ["-Xptxas", "-v"]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(obj)
    failed = []
    for src, p in procs:
        log, _ = p.communicate()
        if p.returncode != 0 or verbose:
            sys.stderr.write(log.decode())
        if p.returncode != 0:
            failed.append(src)
    if failed:
        raise RuntimeError("nvcc failed for: " + ", ".join(failed))
    tmp = target + ".tmp"
    # NCCL (the descriptor all-gather, csrc/comm.cu) is opened at run time
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-o", tmp, *objs, "-ldl"])
    os.replace(tmp, target)
    return target


if __name__ == "__main__":
    args = sys.argv[1:]
    defs = [a for a in args if a.startswith("-D")]
    out = next((a.split("=", 1)[1] for a in args if a.startswith("--out=")), None)
    print(build(force="--force" in args, verbose="-v" in args, defines=defs, out=out))
