"""Build libsdas.so (sm_100a) in-tree with nvcc.  No JIT cache, no CPU fallback."""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("SDAS_LIB", os.path.join(HERE, "libsdas.so"))   # SDAS_LIB: alternate build (debug)
SOURCES = [os.path.join(CSRC, "sdas_kernels.cu"), os.path.join(CSRC, "sdas_host.cpp")]
HEADERS = [os.path.join(CSRC, f) for f in sorted(os.listdir(CSRC)) if f.endswith((".h", ".cuh"))] + \
    [os.path.join(os.path.dirname(HERE), "include", "sdas.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared"]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in SOURCES + HEADERS)


def build(force=False, verbose=False, debug=False, out=None):
    out = out or LIB
    if not force and out == LIB and not needs_build():
        return LIB
    flags = [f for f in FLAGS if f not in ("-O3", "-lineinfo")] + ["-G"] if debug else FLAGS
    extra = os.environ.get("SDAS_NVCC_EXTRA", "").split()   # experiments only (e.g. -DK1_LB_THREADS=128)
    cmd = [NVCC] + flags + extra + (["-Xptxas", "-v"] if verbose else []) + ["-o", out] + SOURCES
    subprocess.check_call(cmd, cwd=HERE)
    return LIB


if __name__ == "__main__":
    dbg = "--debug" in sys.argv
    out = os.path.join(HERE, "libsdas_dbg.so") if dbg else None
    print(build(force="--force" in sys.argv or dbg, verbose="-v" in sys.argv, debug=dbg, out=out))
