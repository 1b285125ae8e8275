"""Build libnc.so in-tree (nvcc, sm_100a) -- the product's CUDA library (include/nc.h)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnc.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nccl_paths():
    try:
        import nvidia.nccl as _n  # torch's bundled NCCL (2.28.x); matches the runtime libnccl.so.2
        base = list(_n.__path__)[0]
    except Exception:
        base = os.path.join(os.path.dirname(os.path.dirname(sys.executable)), "lib", "python3.12", "site-packages",
                            "nvidia", "nccl")
    inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
    if os.path.exists(os.path.join(inc, "nccl.h")) and os.path.exists(os.path.join(lib, "libnccl.so.2")):
        return inc, lib
    return None, None


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "nc.h"), __file__]
    return any(os.path.getmtime(f) > t for f in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    inc, lib = nccl_paths()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--extended-lambda", "-shared", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall",
           "-Xcompiler", "-fopenmp", "-lgomp",
           "-I", os.path.join(ROOT, "include"), "-o", LIB + ".tmp"]
    if inc:
        cmd += ["-DNC_WITH_NCCL=1", "-I", inc, "-L", lib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + lib]
    else:
        cmd += ["-DNC_WITH_NCCL=0"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    cmd += sources()
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
