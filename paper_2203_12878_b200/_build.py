"""Build libmapcheck.so in-tree with nvcc for sm_100a (no GPU needed)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmapcheck.so")

SOURCES = [
    "compiler/front.cpp",
    "compiler/compile.cpp",
    "capi/mapcheck.cpp",
    "capi/jit.cpp",
    "capi/bcapi.cpp",
    "capi/execute.cpp",
    "capi/alloc.cpp",
    "babycuda/bcgen.cpp",
    "babycuda/bcfront.cpp",
    "kernels/generate.cu",
    "kernels/radix.cu",
    "kernels/detect.cu",
    "kernels/rsweep.cu",
    "kernels/exchange.cu",
    "kernels/table.cu",
    "kernels/listing.cu",
    "kernels/direct.cu",
    "kernels/bcexec.cu",
]
HEADERS = ["devabi.h", "compiler/front.h", "compiler/compiler.h", "kernels/common.cuh", "kernels/segstate.cuh",
           "capi/jit.h", "babycuda/bcfront.h", "babycuda/bcgen.h"]

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
    "-Xcompiler", "-fPIC", "-shared",
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "mapcheck.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB + ".tmp", *[os.path.join(CSRC, s) for s in SOURCES], "-lcudart", "-lnvrtc"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
