"""In-tree build of libnumpmp_cuda.so for sm_100a (nvcc, no JIT cache).

    python -m paper_2509_10722_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_DIR = os.path.join(HERE, "lib")
OUT = os.path.join(LIB_DIR, "libnumpmp_cuda.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("pmp_solver.cu", "host_gen.cpp", "host_io.cpp")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in ("pmp_kernels.cuh", "pmp_aux.cuh", "pmp_p2p.cuh",
                                                            "host_instance.h", "host_mt.h")] + [
    os.path.join(ROOT, "include", f) for f in ("numpmp_gpu.h", "numpmp_host.h")
]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(LIB_DIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-o", OUT, *SOURCES,
           "-ldl", "-cudart", "static"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
