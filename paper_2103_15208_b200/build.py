"""Build libcdr.so (the C-ABI of include/cdr.h) in-tree for sm_100a.

    python -m paper_2103_15208_b200.build [--force]

Every .cu under csrc/ is compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo -O3 -fmad=false``
(no FMA contraction: the exactness contract of DESIGN.md §3) and linked with
the static CUDA runtime into paper_2103_15208_b200/lib/libcdr.so.
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
OUT_DIR = os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(PKG, "lib", "obj")
LIB = os.path.join(OUT_DIR, "libcdr.so")
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + ["-O3", "-std=c++17", "-lineinfo", "-fmad=false", "-Xcompiler", "-fPIC",
                "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh")) +
                               glob.glob(os.path.join(CSRC, "*.h")) +
                               [os.path.join(ROOT, "include", "cdr.h")])


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose, obj_dir=None, extra=()):
    obj = os.path.join(obj_dir or OBJ_DIR, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *FLAGS, *extra, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=()) -> str:
    """Compile + link; `out`/`defines` build an experimental variant elsewhere."""
    lib = out or LIB
    obj_dir = OBJ_DIR if out is None else os.path.join(os.path.dirname(out), "obj_" + os.path.basename(out))
    os.makedirs(obj_dir, exist_ok=True)
    if not force and not _stale(lib, _deps()):
        return lib
    extra = [f"-D{d}" for d in defines]
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, obj_dir, extra), _sources()))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    # export exactly the C-ABI (cdr_*); everything else stays local
    vs = os.path.join(obj_dir, "exports.map")
    with open(vs, "w") as f:
        f.write("{ global: cdr_*; local: *; };\n")
    cmd = [NVCC, *ARCH, "-shared", "-o", lib, *objs, "-Xlinker", f"--version-script={vs}", "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return lib


CHECKED_LIB = os.path.join(OUT_DIR, "checked", "libcdr.so")


def build_checked(force: bool = False) -> str:
    """The same library with the device-side bounds checks on (-DCDR_CHECKED,
    CDR_DCHECK in common.cuh): the GPU suite runs against it too
    (tests/test_checked_build.py) in place of compute-sanitizer, which the GPU
    pool does not offer."""
    os.makedirs(os.path.dirname(CHECKED_LIB), exist_ok=True)
    return build(force=force, out=CHECKED_LIB, defines=("CDR_CHECKED",))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
