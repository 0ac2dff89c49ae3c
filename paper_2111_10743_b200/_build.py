"""In-tree build of libb200lb.so (nvcc, sm_100a) and of the oracle's C
library.  Called by __graft_entry__.build(); also runnable directly:

    python -m paper_2111_10743_b200._build
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libb200lb.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-warn-spills", "-Xcompiler", "-fopenmp",
]


def _nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) +
                  glob.glob(os.path.join(CSRC, "*.cpp")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + \
        sorted(glob.glob(os.path.join(CSRC, "*.h"))) + \
        sorted(glob.glob(os.path.join(ROOT, "include", "*.h")))


def needs_build(out=LIB):
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps())


def _obj(src):
    return os.path.join(ROOT, "build", "obj", os.path.basename(src) + ".o")


def build(force=False, verbose=True, extra=()):
    """Compile every source to its own object in parallel (one nvcc per
    translation unit, only the stale ones), then link the shared library."""
    if not force and not needs_build():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    os.makedirs(os.path.join(ROOT, "build", "obj"), exist_ok=True)
    hdr = [d for d in deps() if d not in sources()]
    t_hdr = max(os.path.getmtime(h) for h in hdr)
    flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def stale(src):
        o = _obj(src)
        return force or not os.path.exists(o) or \
            os.path.getmtime(o) < max(os.path.getmtime(src), t_hdr)

    def compile_one(src):
        cmd = [_nvcc(), *flags, *extra, "-I", os.path.join(ROOT, "include"),
               "-c", src, "-o", _obj(src) + ".tmp"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        subprocess.run(cmd, check=True)
        os.replace(_obj(src) + ".tmp", _obj(src))

    todo = [s for s in sources() if stale(s)]
    with ThreadPoolExecutor(max(1, min(len(todo), os.cpu_count() or 1))) as ex:
        list(ex.map(compile_one, todo))
    cmd = [_nvcc(), "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
           "-Xcompiler", "-fopenmp", "-o", LIB + ".tmp", *[_obj(s) for s in sources()], "-lcudart", "-lgomp",
           "-Xlinker", "-rpath=/usr/local/cuda/lib64"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(LIB + ".tmp", LIB)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
