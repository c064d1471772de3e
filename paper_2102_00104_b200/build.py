"""Build the in-tree sm_100a library libttsvd_cu.so (C-ABI: include/ttsvd_cu.h).

``python -m paper_2102_00104_b200.build`` or ``build()``.  nvcc cross-compiles
for sm_100a without a GPU; the .so lands next to this file so it travels to
the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libttsvd_cu.so")
PROBE = os.path.join(HERE, "libttsvd_probe.so")  # bench-only FP64 peak probe
SOURCES = [os.path.join(HERE, "csrc", "ttsvd_cu.cu")]
DEPS = SOURCES + [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))] + [
    os.path.join(ROOT, "include", "ttsvd_cu.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
    "--expt-relaxed-constexpr",
]


def needs_build(out: str = LIB) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(p) > t for p in DEPS if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    for out, srcs in ((LIB, SOURCES), (PROBE, [os.path.join(HERE, "csrc", "probe.cu")])):
        if force or needs_build(out):
            cmd = [NVCC, *FLAGS, "-o", out, *srcs]
            if verbose:
                print(" ".join(cmd), file=sys.stderr)
            subprocess.run(cmd, check=True, cwd=HERE)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
