"""Build the in-tree shared library libgeopairs_b200.so for sm_100a.

    python -m paper_2007_16076_b200.build
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SOURCES = ["propagate.cu", "propagate_cluster.cu", "propagate_big.cu", "commit.cu", "setup.cu", "apgd.cu", "capi.cu"]
OUT = os.path.join(HERE, "libgeopairs_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",  # no FMA contraction: fp32 sums round exactly as the restatement
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def needs_build() -> bool:
    if not os.path.exists(OUT):
        return True
    t = os.path.getmtime(OUT)
    deps = [os.path.join(HERE, "csrc", f) for f in os.listdir(os.path.join(HERE, "csrc"))]
    deps.append(os.path.join(ROOT, "include", "geopairs_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False) -> str:
    if not force and not needs_build():
        return OUT
    srcs = [os.path.join(HERE, "csrc", s) for s in SOURCES]
    extra = os.environ.get("GP_NVCC_EXTRA", "").split()  # dev: tuning -D flags
    cmd = [NVCC, *FLAGS, *extra, "-o", OUT, *srcs]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
