"""In-tree build of libabsp.so (sm_100a) with plain nvcc.

The library is compiled for exactly one target, `-gencode arch=compute_100a,code=sm_100a`;
no fast-math (the centroid/quantizer/scoring kernels reproduce the reference's IEEE
fp32/fp64 op sequences bit for bit). Objects are rebuilt only when a source or
header is newer than the library.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
CSRC = PKG / "csrc"
LIBDIR = PKG / "lib"
LIB = LIBDIR / "libabsp.so"
OBJDIR = ROOT / "build" / "obj"

SOURCES = ["api.cu", "engine.cu", "build_store.cu", "score.cu", "topk.cu", "select.cu", "attend.cu", "dense.cu", "calibrate.cu", "synth.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-Xptxas", "-warn-spills"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def _newest_input() -> float:
    files = list(CSRC.glob("*")) + [ROOT / "include" / "absp.h", Path(__file__)]
    return max(f.stat().st_mtime for f in files if f.is_file())


def build(force: bool = False, verbose: bool = False, trace: bool = False) -> Path:
    """trace=True builds lib/libabsp_trace.so with the attention timeline
    instrumentation (-DABSP_ATTN_TRACE, tools/attn_trace.py); never the product."""
    lib = LIBDIR / "libabsp_trace.so" if trace else LIB
    objdir = OBJDIR.parent / "obj_trace" if trace else OBJDIR
    if lib.exists() and not force and lib.stat().st_mtime >= _newest_input():
        return lib
    objdir.mkdir(parents=True, exist_ok=True)
    LIBDIR.mkdir(parents=True, exist_ok=True)
    # an object is rebuilt when its source, a shared header or this script is newer
    headers = list(CSRC.glob("*.cuh")) + [ROOT / "include" / "absp.h", Path(__file__)]
    newest_header = max(f.stat().st_mtime for f in headers)
    jobs = []
    objs = []
    for src in SOURCES:
        obj = objdir / (Path(src).stem + ".o")
        objs.append(str(obj))
        if (not force and obj.exists()
                and obj.stat().st_mtime >= max(newest_header, (CSRC / src).stat().st_mtime)):
            continue
        cmd = [nvcc(), *ARCH, *FLAGS, *(["-DABSP_ATTN_TRACE"] if trace else []),
               *os.environ.get("ABSP_EXTRA_NVCC", "").split(), "-I", str(ROOT / "include"),
               "-I", str(CSRC), "-c", str(CSRC / src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), file=sys.stderr)
        jobs.append(cmd)
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4) or 1) as ex:
        for r in list(ex.map(lambda c: subprocess.run(c, check=True), jobs)):
            pass
    tmp = lib.with_suffix(".so.tmp")
    cmd = [nvcc(), *ARCH, "-shared", "-o", str(tmp), *objs, "-lcudart_static", "-lrt", "-ldl", "-lpthread"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, trace="--trace" in sys.argv))
