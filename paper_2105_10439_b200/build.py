"""Build the native library in-tree for sm_100a.

    python -m paper_2105_10439_b200.build [--force]

nvcc cross-compiles without a GPU, so this runs in the CPU build container;
the resulting ``_lib/libcofem_b200.so`` travels with the repo snapshot.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libcofem_b200.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_include():
    try:
        import nvidia.nccl  # type: ignore

        base = os.path.dirname(nvidia.nccl.__file__) if nvidia.nccl.__file__ else list(nvidia.nccl.__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except Exception:
        pass
    for cand in ("/usr/include", "/usr/local/include"):
        if os.path.exists(os.path.join(cand, "nccl.h")):
            return cand
    raise RuntimeError("nccl.h not found (needed for the NCCL type declarations)")


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.exists(cand) or cand == "nvcc"):
            return cand
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "cofem_b200.h")])


def up_to_date():
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(s) <= t for s in sources())


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
           "-I", os.path.join(ROOT, "include"), "-I", _nccl_include(),
           os.path.join(CSRC, "cofem.cu"), "-o", OUT + ".tmp", "-ldl", "-lpthread"]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
