"""Build libgps.so (all CUDA sources, sm_100a) in-tree with nvcc.

    python paper_2509_11574_b200/build.py [--force]   (no package import: works before libgps.so exists)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgps.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-Xcompiler", "-ffp-contract=off", "--expt-relaxed-constexpr",
         "-diag-suppress", "177,550", f"-I{os.path.join(ROOT, 'include')}"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(ROOT, "include", "gps.h")]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in deps())


LIB_CHECKED = os.path.join(HERE, "libgps_checked.so")


def build(force: bool = False, verbose: bool = False, out: str | None = None, checked: bool = False) -> str:
    """checked=True: the bounds-checked variant (-DGPS_CHECKED) into
    libgps_checked.so (or `out`); the production library is never replaced by it."""
    if checked and out is None:
        out = LIB_CHECKED
    if out is None and not force and up_to_date():
        return LIB
    objs = []
    bdir = os.path.join(HERE, "build_checked" if checked else "build")
    os.makedirs(bdir, exist_ok=True)
    procs = []
    for src in sources():
        obj = os.path.join(bdir, os.path.basename(src)[:-3] + ".o")
        cmd = [NVCC, *FLAGS, *(["-DGPS_CHECKED"] if checked else []), "-c", src, "-o", obj]
        if verbose:
            print(" ".join(cmd))
        procs.append(subprocess.Popen(cmd))
        objs.append(obj)
    for p in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, p.args)
    dst = out or LIB
    os.makedirs(os.path.dirname(os.path.abspath(dst)), exist_ok=True)
    tmp = dst + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", *objs,
                           "-o", tmp, "-lcudart"])
    os.replace(tmp, dst)
    return dst


if __name__ == "__main__":
    # --out PATH: build the current tree into PATH (A/B experiments, tools/ab.sh) instead of libgps.so
    o = sys.argv[sys.argv.index("--out") + 1] if "--out" in sys.argv else None
    print(build(force="--force" in sys.argv, verbose=True, out=o, checked="--checked" in sys.argv))
