"""Build liblhaf.so in-tree: the sm_100a kernels + the C++ host library behind include/lhaf.h.

    python -m paper_2108_01622_b200.build          (or __graft_entry__.build())

nvcc cross-compiles for sm_100a without a GPU.  The .so is git-ignored but travels to the GPU
box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "liblhaf.so")
SOURCES = [os.path.join(CSRC, f) for f in ("lhaf_kernels.cu", "lhaf_v3.cu", "lhaf_v5.cu", "lhaf_tree.cu", "lhaf_host.cpp", "lhaf_gbs.cpp")]
HEADERS = [os.path.join(CSRC, "lhaf_internal.h"), os.path.join(CSRC, "lhaf_device.cuh"), os.path.join(CSRC, "lhaf_tail.cuh"), os.path.join(ROOT, "include", "lhaf.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False, out: str | None = None) -> str:
    """Compile liblhaf.so (or a diagnostic variant at `out`; LHAF_NVCC_EXTRA adds nvcc flags)."""
    target = out or LIB
    if out is None and not force and not _stale():
        return LIB
    extra = os.environ.get("LHAF_NVCC_EXTRA", "").split()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", *extra,
           "-Xptxas", "-v" if verbose else "-O3", "-shared", "-o", target, *SOURCES,
           "-I", os.path.join(ROOT, "include"), "-ldl"]
    subprocess.check_call(cmd)
    if out is not None:
        return target
    pkg = sys.modules.get("paper_2108_01622_b200")
    if pkg is not None and hasattr(pkg, "reload_library"):
        try:  # a stale copy already mapped in this process cannot be replaced; new processes load the new one
            pkg.reload_library()
        except (OSError, AttributeError):
            pass
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
