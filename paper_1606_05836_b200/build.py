"""Build libpermb200.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

    python -m paper_1606_05836_b200.build [--force] [-j N]

Each csrc/perm_inst_*.cu instantiates one template per n for a range of n, so the
translation units compile in parallel; perm_api.cu holds the C ABI.
"""
from __future__ import annotations

import argparse
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libpermb200.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--fmad=true", f"-I{INCLUDE}",
         "-Xptxas", "-warn-spills"]


def _deps() -> list[str]:
    return glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(INCLUDE, "permb200.h")]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _compile(src: str, verbose: bool, build_dir: str = BUILD, extra=()) -> tuple[str, str]:
    obj = os.path.join(build_dir, os.path.basename(src)[:-3] + ".o")
    if not _stale(obj, [src] + _deps()):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, *extra, "-c", src, "-o", obj + ".tmp"]
    if verbose:
        cmd += ["-Xptxas", "-v"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj, r.stderr


CHECKED_LIB = os.path.join(HERE, "libpermb200_checked.so")


def build(force: bool = False, jobs: int | None = None, verbose: bool = False, checked: bool = False) -> str:
    """checked=True: the bounds-checked debug build (-DPERMB200_CHECKED: device-side checks of
    every shared-memory / table index, trap on failure) -> libpermb200_checked.so, loaded with
    PERMB200_LIB=<path> (compute-sanitizer is not available on the GPU pool)."""
    build_dir = BUILD + ("_checked" if checked else "")
    lib = CHECKED_LIB if checked else LIB
    extra = ("-DPERMB200_CHECKED",) if checked else ()
    os.makedirs(build_dir, exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    if force:
        for o in glob.glob(os.path.join(build_dir, "*.o")):
            os.remove(o)
    jobs = jobs or max(1, min(len(srcs), os.cpu_count() or 1))
    logs = []
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = []
        for obj, log in ex.map(lambda s: _compile(s, verbose, build_dir, extra), srcs):
            objs.append(obj)
            if log:
                logs.append(log)
    if force or _stale(lib, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", lib + ".tmp", *objs, "-cudart=static"]
        subprocess.run(cmd, check=True)
        os.replace(lib + ".tmp", lib)
    LIB_OUT = lib
    if verbose:
        sys.stderr.write("\n".join(logs))
    return LIB_OUT


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    ap.add_argument("-j", type=int, default=None)
    ap.add_argument("-v", "--verbose", action="store_true")
    ap.add_argument("--checked", action="store_true", help="bounds-checked debug build")
    a = ap.parse_args()
    print(build(a.force, a.j, a.verbose, a.checked))
