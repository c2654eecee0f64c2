"""Compile libqaprlt2.so (sm_100a) in-tree with nvcc.

The library is the C ABI of include/qap_rlt2.h: kernels (csrc/rlt2_kernels.cu) and host
control (csrc/rlt2_host.cu).  cudart is linked statically so the .so only needs the
driver at run time.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libqaprlt2.so")
SOURCES = [os.path.join(HERE, "csrc", f) for f in ("rlt2_kernels.cu", "rlt2_host.cu", "rlt2_shard.cu")]
HEADERS = [os.path.join(HERE, "csrc", f) for f in ("rlt2_internal.h", "rlt2_shard.h")] + \
          [os.path.join(ROOT, "include", "qap_rlt2.h")]


def nccl_include():
    """NCCL headers matching torch's bundled libnccl (nvidia-nccl wheel), if present."""
    try:
        import nvidia.nccl
        for base in nvidia.nccl.__path__:
            inc = os.path.join(base, "include")
            if os.path.exists(os.path.join(inc, "nccl.h")):
                return inc
    except Exception:
        pass
    return "/usr/include" if os.path.exists("/usr/include/nccl.h") else None
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-fmad=false", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(f) > t for f in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    inc = nccl_include()
    nccl = ["-DQAP_HAVE_NCCL", "-I", inc] if inc else []
    cmd = [NVCC, *FLAGS, *nccl, *(["-Xptxas", "-v"] if verbose else []), "-o", tmp, *SOURCES, "-ldl"]
    subprocess.check_call(cmd, cwd=ROOT)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
