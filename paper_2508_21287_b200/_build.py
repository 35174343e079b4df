"""Build libdeltamotif.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libdeltamotif.so")
# checked variant: device bounds checks (DM_DCHECK, -DDM_CHECKED) trap on a bad index; loaded
# when DM_LIBRARY_VARIANT=checked (tests/test_gpu_checked.py)
LIB_CHECKED = os.path.join(PKG, "libdeltamotif_checked.so")
SOURCES = ["errors.cpp", "planner.cpp", "graph.cu", "extend.cu", "tail.cu", "pairs.cu", "apex.cu", "exchange.cu", "tabstep.cu", "motifdb.cu", "scoring.cu", "match.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3,-fvisibility=hidden",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", CSRC]


def _stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(ROOT, "include", "deltamotif.h")]
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(force: bool, verbose: bool, checked: bool):
    """Start one nvcc per stale translation unit of a variant; returns (lib, objs, procs)."""
    lib = LIB_CHECKED if checked else LIB
    objdir = os.path.join(PKG, "build_checked" if checked else "build")
    os.makedirs(objdir, exist_ok=True)
    headers = [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".h", ".cuh"))]
    headers.append(os.path.join(ROOT, "include", "deltamotif.h"))
    newest_hdr = max(os.path.getmtime(h) for h in headers)
    flags = FLAGS + (["-DDM_CHECKED"] if checked else [])
    objs, procs = [], []
    for src in SOURCES:  # one nvcc per translation unit, in parallel; stale objects only
        obj = os.path.join(objdir, src + ".o")
        objs.append(obj)
        spath = os.path.join(CSRC, src)
        if (not force and os.path.exists(obj)
                and os.path.getmtime(obj) > max(os.path.getmtime(spath), newest_hdr)):
            continue
        cmd = [NVCC, *ARCH, *flags, "-c", spath, "-o", obj + ".tmp"]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        procs.append((subprocess.Popen(cmd), obj))
    return lib, objs, procs


def _link(lib: str, objs, procs):
    for p, obj in procs:
        if p.wait() != 0:
            raise subprocess.CalledProcessError(p.returncode, "nvcc")
        os.replace(obj + ".tmp", obj)
    tmp = lib + f".tmp{os.getpid()}"
    subprocess.check_call([NVCC, *ARCH, "-shared", *objs, "-o", tmp])
    os.replace(tmp, lib)
    return lib


def build(force: bool = False, verbose: bool = False, checked: bool = False) -> str:
    """libdeltamotif.so, or with checked=True libdeltamotif_checked.so (-DDM_CHECKED)."""
    lib = LIB_CHECKED if checked else LIB
    if not force and not _stale(lib):
        return lib
    return _link(*_compile(force, verbose, checked))


def build_all(force: bool = False, verbose: bool = False):
    """Both variants, every translation unit of both compiling concurrently."""
    jobs = [_compile(force, verbose, chk) for chk in (False, True)
            if force or _stale(LIB_CHECKED if chk else LIB)]
    return [_link(*j) for j in jobs]


if __name__ == "__main__":
    if "--all" in sys.argv:
        print(build_all(force="--force" in sys.argv, verbose=True))
    else:
        print(build(force="--force" in sys.argv, verbose=True, checked="--checked" in sys.argv))
