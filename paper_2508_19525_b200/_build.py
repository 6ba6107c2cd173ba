"""Build libblb.so in-tree: nvcc for sm_100a (CUDA kernels + C ABI) and g++ for
the host table generator (needs libquadmath)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libblb.so")
# compile-time kernel variants for A/B measurements are separate files: build(defines=[...], out=path)
ROOT = os.path.dirname(HERE)

CU = ["ntt.cu", "kernels.cu", "encode.cu", "matmul.cu", "qk.cu", "api.cu", "peaks.cu"]
CPP = ["host_tables.cpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return [os.path.join(CSRC, f) for f in CU + CPP] + [os.path.join(CSRC, "blb_internal.cuh"),
                                                       os.path.join(ROOT, "include", "blb.h")]


def needs_build() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """defines: extra -D flags (kernel tuning variants, e.g. BLB_NTT_MINB=3); out: alternative .so path."""
    so = out or SO
    if not force and not defines and out is None and not needs_build():
        return SO
    bdir = os.path.join(HERE, "build" if not defines else "build_" + "_".join(d.replace("=", "") for d in defines))
    os.makedirs(bdir, exist_ok=True)
    objs = []
    for f in CPP:
        o = os.path.join(bdir, f + ".o")
        subprocess.check_call(["g++", "-O2", "-fPIC", "-std=gnu++17", "-fext-numeric-literals", "-c", os.path.join(CSRC, f), "-o", o])
        objs.append(o)
    for f in CU:
        o = os.path.join(bdir, f + ".o")
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
               *["-D" + d for d in defines], "-I", os.path.join(ROOT, "include"), "-c", os.path.join(CSRC, f), "-o", o]
        subprocess.check_call(cmd)
        objs.append(o)
    tmp = so + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lquadmath", "-lcudart"])
    os.replace(tmp, so)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
