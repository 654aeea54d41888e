"""Build librbf.so (the C-ABI of include/rbf.h) in-tree with nvcc for sm_100a.

    python -m paper_1305_5179_b200.build [--force]     # or __graft_entry__.build()

Each csrc/*.cu compiles to its own object (in parallel, under build/), then one
nvcc -shared link.  An object is rebuilt when its source, any csrc/*.h or
include/rbf.h is newer than it.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "librbf.so")
OBJDIR = os.path.join(HERE, "build")
# the CHECKED build (csrc/checks.h: device bounds checks + lane/warp jitter at the
# shared-memory hand-over points; tools/race_probe.py, tests/test_gpu_race_probe.py)
LIB_CHECKED = os.path.join(HERE, "librbf_checked.so")
OBJDIR_CHECKED = os.path.join(HERE, "build_checked")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++20", "-Xcompiler", "-fPIC,-ffp-contract=off",
          "-diag-suppress", "177"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.h"))) + [os.path.join(ROOT, "include", "rbf.h")]


def deps():
    return sources() + headers()


def _obj(src: str, objdir: str = OBJDIR) -> str:
    return os.path.join(objdir, os.path.basename(src)[:-3] + ".o")


def up_to_date(lib: str = LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(p) <= t for p in deps())


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    lib, objdir = (LIB_CHECKED, OBJDIR_CHECKED) if checked else (LIB, OBJDIR)
    flags = CFLAGS + (["-DRBF_CHECKED"] if checked else [])
    if not force and up_to_date(lib):
        return lib
    os.makedirs(objdir, exist_ok=True)
    th = max(os.path.getmtime(h) for h in headers())
    todo = [s for s in sources()
            if force or not os.path.exists(_obj(s, objdir))
            or os.path.getmtime(_obj(s, objdir)) < max(th, os.path.getmtime(s))]

    def compile_one(src):
        cmd = [NVCC, *flags, "-c", "-o", _obj(src, objdir) + ".tmp", src]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.run(cmd, check=True)
        os.replace(_obj(src, objdir) + ".tmp", _obj(src, objdir))

    with ThreadPoolExecutor(max_workers=max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, todo))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *[_obj(s, objdir) for s in sources()]]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
