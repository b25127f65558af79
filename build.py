"""Build the native pieces in-tree.

  paper_1102_0183_b200/libckb200.so   CUDA engine + C ABI (sm_100a)
  oracle/liboracle.so                 CPU oracle (test infrastructure)

    python build.py            # both
    python build.py --cuda     # engine only
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_1102_0183_b200")
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libckb200.so")
SOURCES = ["ck_seam.cu", "ck_net.cu", "ck_deform.cu", "ck_tc.cu", "ck_tct.cu"]
HEADERS = ["ck_numerics.cuh", "ck_engine.cuh", "ck_kernels.cuh", "ck_host.h", "ck_specs.inc",
           "ck_tc_common.cuh"]

COMPILE_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-I", os.path.join(ROOT, "include"),
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared"]
# per-unit extras: the tensor-core GEMMs run at register caps set by their
# launch bounds (3-4 CTAs per SM); a spill there must fail the build
UNIT_FLAGS = {"ck_tc.cu": ["-Xptxas=-warn-spills,-Werror"],
              "ck_tct.cu": ["-Xptxas=-warn-spills,-Werror"]}


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


SPECS = os.path.join(CSRC, "ck_specs.inc")


def _spec_units() -> list[str]:
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)
                  if f.startswith("ck_spec_") and f.endswith(".cu"))


OBJ_DIR = os.path.join(ROOT, "build", "obj")


def _compile(out: str, verbose: bool, extra=(), specs: bool = True) -> None:
    """Every translation unit to an object in parallel, then one link.
    Objects are cached under build/obj (per flag set) and recompiled only when
    the unit or a shared header changed."""
    units = [os.path.join(CSRC, s) for s in SOURCES] + (_spec_units() if specs else [])
    headers = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include",
                                                                      "ckb200.h")]
    tag = "stage1" if "-DCK_NO_SPECS" in extra else "full"
    odir = os.path.join(OBJ_DIR, tag)
    os.makedirs(odir, exist_ok=True)
    procs = []
    objs = []
    for u in units:
        obj = os.path.join(odir, os.path.basename(u) + ".o")
        objs.append(obj)
        if not verbose and not _stale(obj, [u, *headers, __file__]):
            continue
        cmd = [_nvcc(), *COMPILE_FLAGS, *extra, *UNIT_FLAGS.get(os.path.basename(u), []),
               "-c", "-o", obj, u]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        procs.append((obj, subprocess.Popen(cmd)))
    for obj, p in procs:
        if p.wait() != 0:
            if os.path.exists(obj):
                os.remove(obj)
            raise subprocess.CalledProcessError(p.returncode, "nvcc")
    subprocess.run([_nvcc(), *LINK_FLAGS, "-o", out, *objs], check=True)


def generate_specs(lib: str) -> bool:
    """Regenerate ck_specs.inc (+ ck_spec_*.cu) with `lib`'s geometry builder."""
    before = open(SPECS).read() if os.path.exists(SPECS) else None
    subprocess.run([sys.executable, os.path.join(ROOT, "tools", "gen_specs.py"), lib, SPECS],
                   check=True)
    return open(SPECS).read() != before


def build_cuda(force: bool = False, verbose: bool = False) -> str:
    """Two stages: a library without specialised kernels (its geometry builder
    prints ck_specs.inc and one ck_spec_<net>.cu per BASELINE net), then the
    full library."""
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "ckb200.h"))
    deps.append(os.path.join(ROOT, "paper_1102_0183_b200", "configs.py"))
    deps.remove(SPECS)
    if force or _stale(LIB, deps):
        # stage 1: the library without specialised kernels generates the specs
        stage1 = os.path.join(PKG, "libckb200_stage1.so")
        _compile(stage1, False, ["-DCK_NO_SPECS"], specs=False)
        generate_specs(stage1)
        os.remove(stage1)
        # stage 2: the library with them
        _compile(LIB, verbose)
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
