"""Build libpbicgstab.so (sm_100a) in-tree with nvcc.

Flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo (ncu source
view), -fmad=false (no implicit contraction: every FMA on the value path is an
explicit __fma_rn, FMA policy F of DESIGN.md), no fast-math (IEEE div/sqrt).
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.environ.get("PBCG_LIB") or os.path.join(HERE, "libpbicgstab.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def nccl_include() -> str:
    try:
        import nvidia.nccl  # type: ignore
        d = os.path.join(list(nvidia.nccl.__path__)[0], "include")
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    except Exception:
        pass
    for d in ("/usr/include",):
        if os.path.exists(os.path.join(d, "nccl.h")):
            return d
    raise RuntimeError("nccl.h not found")


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cuh"))
                  + [os.path.join(ROOT, "include", "pbicgstab.h")])


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    target = out or LIB
    if out is None and not force and not needs_build():
        return LIB
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
           "-fmad=false", "-Xcompiler", "-fPIC,-O2", "-shared",
           "-I", os.path.join(ROOT, "include"), "-I", nccl_include(),
           "-o", target + ".tmp", os.path.join(CSRC, "runtime.cu"), "-ldl", "-lcudart"] + [f"-D{d}" for d in defines]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    print("[build]", " ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(target + ".tmp", target)
    return target


if __name__ == "__main__":
    if "--variant" in sys.argv:  # python build.py --variant NAME DEFINE...
        i = sys.argv.index("--variant")
        build(force=True, out=os.path.join(HERE, f"libpbicgstab_{sys.argv[i + 1]}.so"), defines=tuple(sys.argv[i + 2:]))
    elif "--debug-counters" in sys.argv:
        build(force=True, verbose="-v" in sys.argv, out=os.path.join(HERE, "libpbicgstab_dbg.so"),
              defines=("PBCG_DEBUG_COUNTERS",))
    else:
        build(force="--force" in sys.argv, verbose="-v" in sys.argv)
