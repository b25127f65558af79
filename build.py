"""Build the native pieces in-tree.

  paper_1102_0183_b200/libckb200.so   CUDA engine + C ABI (sm_100a)
  oracle/liboracle.so                 CPU oracle (test infrastructure)

    python build.py            # both
    python build.py --cuda     # engine only
"""

from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1102_0183_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libckb200.so")
SOURCES = ["ck_seam.cu", "ck_net.cu"]
HEADERS = ["ck_numerics.cuh", "ck_engine.cuh", "ck_host.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-I", os.path.join(ROOT, "include"),
]


def _nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _stale(target: str, deps: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "ckb200.h"))
    if force or _stale(LIB, deps):
        cmd = [_nvcc(), *NVCC_FLAGS, "-o", LIB, *[os.path.join(CSRC, s) for s in SOURCES]]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
    return LIB


def build_oracle(force: bool = False) -> str:
    args = ["make", "-s", "-C", os.path.join(ROOT, "oracle")]
    if force:
        args.append("-B")
    subprocess.run(args, check=True)
    return os.path.join(ROOT, "oracle", "liboracle.so")


def main(argv: list[str]) -> None:
    force = "--force" in argv
    verbose = "-v" in argv
    if "--oracle" not in argv:
        print(build_cuda(force, verbose))
    if "--cuda" not in argv:
        print(build_oracle(force))


if __name__ == "__main__":
    main(sys.argv[1:])
