"""Build libsdattn.so (sm_100a) in-tree with nvcc.

    python -m paper_2605_24168_b200.build [--force] [--debug]

Each csrc/*.cu is compiled with `-gencode arch=compute_100a,code=sm_100a`
(the explicit `a` target is required for tcgen05/TMA/griddepcontrol PTX) into
build/*.o, then linked into paper_2605_24168_b200/libsdattn.so with the CUDA
runtime linked statically.  Objects are rebuilt when a source or header is
newer than them.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
BUILD = os.path.join(ROOT, "build", "sdattn")
LIB = os.path.join(PKG, "libsdattn.so")
GENCODE = "-gencode=arch=compute_100a,code=sm_100a"


def nvcc_path() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: cannot build the sm_100a library")


def _flags(debug: bool):
    f = ["-std=c++17", GENCODE, "-lineinfo", "-Xcompiler", "-fPIC", "-I", INCLUDE, "-I", CSRC,
         "--expt-relaxed-constexpr", "--extended-lambda", "-Xptxas", "-v"]
    f += ["-O0", "-G"] if debug else ["-O3"]
    f += os.environ.get("SD_NVCC_EXTRA", "").split()  # build-time variants (A/B experiments)
    return f


def _stale(obj: str, src: str, headers) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(p) > t for p in [src, *headers])


def build_library(force: bool = False, debug: bool = False, verbose: bool = False) -> str:
    nvcc = nvcc_path()
    os.makedirs(BUILD, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    headers = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(INCLUDE, "*.h"))
    objs, jobs = [], []
    for s in srcs:
        o = os.path.join(BUILD, os.path.basename(s)[:-3] + ".o")
        objs.append(o)
        if force or _stale(o, s, headers):
            jobs.append((s, o))

    def compile_one(so):
        s, o = so
        cmd = [nvcc, *_flags(debug), "-c", s, "-o", o]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {s}:\n{r.stderr}")
        # keep the ptxas resource report beside the object (registers / spills)
        with open(o + ".ptxas.txt", "w") as fh:
            fh.write(r.stderr)
        return s

    if jobs:
        with cf.ThreadPoolExecutor(max_workers=min(8, len(jobs))) as ex:
            for s in ex.map(compile_one, jobs):
                if verbose:
                    print("compiled", os.path.relpath(s, ROOT))
    if jobs or not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [nvcc, GENCODE, "-shared", "-Xcompiler", "-fPIC", "-cudart", "static", *objs, "-o", LIB]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        if verbose:
            print("linked", os.path.relpath(LIB, ROOT))
    return LIB


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("--debug", action="store_true")
    a = ap.parse_args(argv)
    print(build_library(force=a.force, debug=a.debug, verbose=True))


if __name__ == "__main__":
    sys.exit(main())
