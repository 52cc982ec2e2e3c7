"""Build libragb.so (CUDA kernels for sm_100a + host C++ + C-ABI) in-tree.

    python -m paper_2511_03475_b200.build [--force] [--verbose] [--debug]
        [--variant NAME -DMACRO ...]

Each source compiles to its own object (in parallel; only stale objects are
rebuilt), then one nvcc link produces lib/libragb.so.  --variant builds
lib/libragb_NAME.so with extra -D flags (A/B experiments; load it with
RAGB_LIB=NAME).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIBDIR = os.path.join(PKG, "lib")
OBJDIR = os.path.join(PKG, "build")
LIB = os.path.join(LIBDIR, "libragb.so")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "--fmad=false",                      # parity: no contraction anywhere (X6)
    "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden,-fopenmp",
]
LINK_FLAGS = ["-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-Xcompiler", "-fopenmp", "-lgomp"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(INCLUDE, "ragb.h"), __file__]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False, debug: bool = False, variant: str | None = None,
          defines=()) -> str:
    """debug=True builds lib/libragb_debug.so with device bounds checks
    (-DRAGB_DEBUG); load it with RAGB_LIB=debug."""
    tag = "debug" if debug else variant
    lib = LIB if not tag else os.path.join(LIBDIR, f"libragb_{tag}.so")
    extra = (["-DRAGB_DEBUG"] if debug else []) + list(defines)
    objdir = os.path.join(OBJDIR, tag or "release")
    os.makedirs(objdir, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    nvcc = os.environ.get("NVCC", "nvcc")
    hdrs = _headers()
    jobs = []
    for src in sources():
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        if force or _stale(obj, [src] + hdrs):
            cmd = [nvcc] + NVCC_FLAGS + (["-Xptxas", "-v"] if verbose else []) + extra + \
                ["-I", INCLUDE, "-I", CSRC, "-c", src, "-o", obj + ".tmp"]
            jobs.append((cmd, obj))
    with cf.ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 4))) as ex:
        for (cmd, obj), fut in zip(jobs, [ex.submit(subprocess.check_call, cmd) for cmd, _ in jobs]):
            fut.result()
            os.replace(obj + ".tmp", obj)
    objs = [os.path.join(objdir, os.path.basename(s) + ".o") for s in sources()]
    if jobs or force or _stale(lib, objs):
        subprocess.check_call([nvcc] + LINK_FLAGS + ["-o", lib + ".tmp"] + objs)
        os.replace(lib + ".tmp", lib)
    return lib


if __name__ == "__main__":
    args = sys.argv[1:]
    variant = args[args.index("--variant") + 1] if "--variant" in args else None
    defs = [a for a in args if a.startswith("-D")]
    print(build(force="--force" in args, verbose="--verbose" in args, debug="--debug" in args,
                variant=variant, defines=defs))
