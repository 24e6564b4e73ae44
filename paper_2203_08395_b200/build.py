"""Build libhf.so in-tree with nvcc for sm_100a (no torch extension machinery).

    python -m paper_2203_08395_b200.build [--force]
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libhf.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# no --use_fast_math: IEEE adds, no flush-to-zero (reading R9/R10)
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-ftz=false", "-prec-div=true", "-prec-sqrt=true"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(os.path.dirname(HERE), "include", "hf.h")]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in sources() + headers())


def build(force: bool = False, verbose: bool = False, out: str = None, tag: str = "") -> str:
    """out / tag: an alternative build (e.g. HF_NVCC_FLAGS=-DW1_NU_OVR=4) written next to
    libhf.so for A/B timing through HF_LIB; the default build is libhf.so."""
    lib = out or LIB
    if not force and not out and not stale():
        return LIB
    objdir = os.path.join(HERE, "build" + (("_" + tag) if tag else ""))
    os.makedirs(objdir, exist_ok=True)
    objs = []
    procs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        extra = os.environ.get("HF_NVCC_FLAGS", "").split()
        cmd = [NVCC, *ARCH, *FLAGS, *extra, "-I", os.path.join(os.path.dirname(HERE), "include"),
               "-c", src, "-o", obj]
        procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                            stderr=subprocess.STDOUT, text=True)))
    failed = False
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            failed = True
            sys.stderr.write(f"--- nvcc failed on {src}\n{out}\n")
        elif verbose:
            sys.stderr.write(out)
    if failed:
        raise RuntimeError("nvcc build of libhf.so failed")
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-Xcompiler", "-fPIC", "-o", tmp, *objs,
                           "-ldl", "-lpthread"])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    # python -m paper_2203_08395_b200.build [--force] [-v] [--variant NAME]
    #   --variant NAME: build libhf_NAME.so with $HF_NVCC_FLAGS (A/B through HF_LIB)
    if "--variant" in sys.argv:
        tag = sys.argv[sys.argv.index("--variant") + 1]
        print(build(force=True, verbose="-v" in sys.argv,
                    out=os.path.join(HERE, f"libhf_{tag}.so"), tag=tag))
    else:
        print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
