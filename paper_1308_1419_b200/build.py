"""Build libtrigrid_b200.so in-tree with nvcc for sm_100a.

    python -m paper_1308_1419_b200.build

The shared library is the product: CUDA kernels + the extern "C" ABI of
include/trigrid_b200.h.  It is built in-tree (git-ignored) so it travels to
the GPU box with the repo snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libtrigrid_b200.so")
SOURCES = [os.path.join(CSRC, "trigrid_b200.cu")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("tg_kernels.cuh", "tg_mapping.cuh", "tg_gram.cuh")] + [
    os.path.join(ROOT, "include", "trigrid_b200.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=default",
    "-Xptxas", "-v",
    "--expt-relaxed-constexpr",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in DEPS)


def build(force: bool = False, verbose: bool = False, variant: str | None = None,
          defines: tuple = ()) -> str:
    """Build the library; `variant` + `defines` build an A/B copy
    (libtrigrid_b200_<variant>.so) used only through TG_LIB_PATH."""
    lib = LIB if variant is None else os.path.join(HERE, f"libtrigrid_b200_{variant}.so")
    if not force and variant is None and up_to_date():
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, *[f"-D{d}" for d in defines], "-I", os.path.join(ROOT, "include"),
           "-o", lib + ".tmp", *SOURCES]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libtrigrid_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    if variant is None:
        with open(os.path.join(HERE, "ptxas_report.txt"), "w") as f:
            f.write(res.stderr)
    os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    if "--variant" in sys.argv:
        k = sys.argv.index("--variant")
        name, defs = sys.argv[k + 1], tuple(sys.argv[k + 2:])
        print(build(force=True, variant=name, defines=defs))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
        print(LIB)
