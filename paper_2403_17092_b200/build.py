"""Build libgnnstep.so (sm_100a) in-tree with nvcc.  Used by __graft_entry__.build() and
the binding (which builds on first import if the library is missing or stale)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgnnstep.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dirs():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    roots = list(spec.submodule_search_locations) if spec else []
    for r in roots:
        inc, lib = os.path.join(r, "nccl", "include"), os.path.join(r, "nccl", "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    raise RuntimeError("torch-bundled NCCL (nvidia/nccl) not found")


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
    deps.append(os.path.join(os.path.dirname(HERE), "include", "gnnstep.h"))
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """out/defines: an experiment variant (extra -D flags) built to another path."""
    if out is None and not force and not _stale():
        return LIB
    nccl_inc, nccl_lib = _nccl_dirs()
    target = out or LIB
    objdir = os.path.join(HERE, "build") if out is None else out + ".objs"
    os.makedirs(objdir, exist_ok=True)
    common = ["nvcc", *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
              "-I", nccl_inc, "-I", os.path.join(os.path.dirname(HERE), "include"),
              "-Xptxas", "-v" if verbose else "-O3", *[f"-D{d}" for d in defines]]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        r = subprocess.run(common + ["-c", src, "-o", obj], capture_output=True, text=True)
        if r.returncode:
            raise RuntimeError(f"nvcc failed on {src}:\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    with ThreadPoolExecutor(max_workers=8) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = target + f".{os.getpid()}.tmp"
    r = subprocess.run(["nvcc", *ARCH, "-shared", "-o", tmp, *objs, "-L", nccl_lib, "-l:libnccl.so.2",
                        "-Xlinker", "-rpath=" + nccl_lib, "-lcudart"], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, target)
    return target


HOST_SRC = os.path.join(HERE, "host", "gnnhost.cpp")
HOST_LIB = os.path.join(HERE, "libgnnhost.so")


def build_host(force: bool = False) -> str:
    """libgnnhost.so: the host-core trainer rank (include/gnnhost.h), g++ -O3 -fopenmp.
    -ffp-contract=off: the arithmetic is the source's (the update's fma is explicit)."""
    inc = os.path.join(os.path.dirname(HERE), "include", "gnnhost.h")
    if not force and os.path.exists(HOST_LIB) and all(os.path.getmtime(d) <= os.path.getmtime(HOST_LIB)
                                                      for d in (HOST_SRC, inc)):
        return HOST_LIB
    tmp = HOST_LIB + f".{os.getpid()}.tmp"
    r = subprocess.run(["g++", "-O3", "-std=c++17", "-fopenmp", "-ffp-contract=off", "-fPIC", "-shared",
                        "-I", os.path.dirname(inc), "-o", tmp, HOST_SRC], capture_output=True, text=True)
    if r.returncode:
        raise RuntimeError(f"g++ failed on {HOST_SRC}:\n{r.stderr}")
    os.replace(tmp, HOST_LIB)
    return HOST_LIB


if __name__ == "__main__":
    # python build.py [--force] [-v] [--out PATH -DNAME=VAL ...]  (variants for A/B experiments)
    a = sys.argv[1:]
    o = a[a.index("--out") + 1] if "--out" in a else None
    print(build(force="--force" in a, verbose="-v" in a, out=o, defines=[x[2:] for x in a if x.startswith("-D")]))
