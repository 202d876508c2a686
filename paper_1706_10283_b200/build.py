"""Build libbolt.so in-tree: every csrc/*.cu compiled for sm_100a with nvcc,
linked into paper_1706_10283_b200/libbolt.so (static cudart, C ABI only).

    python -m paper_1706_10283_b200.build [--force] [--verbose]
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
OBJ = os.path.join(PKG, "build")
LIB = os.path.join(PKG, "libbolt.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-O3", "-std=c++17", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-O2,-fvisibility=hidden",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "bolt.h")]


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose, objdir=OBJ):
    obj = os.path.join(objdir, os.path.basename(src)[:-3] + ".o")
    hdrs = glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(ROOT, "include", "bolt.h")]
    if not _stale(obj, [src] + hdrs):
        return obj, ""
    cmd = [NVCC, *NVCC_FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, profile: bool = False, xmode: bool = False,
          variant: str = "") -> str:
    """Diagnostic builds (tools/ only, loaded with BOLT_LIB=<name>):
    profile=True -> libbolt_prof.so with -DBOLT_PROFILE (cycle counters) and -DBOLT_XMODE;
    xmode=True -> libbolt_x.so with -DBOLT_XMODE (BOLT_TC_XMODE experiment
    switches that skip pipeline stages; results are wrong by design)."""
    global NVCC_FLAGS
    lib, objdir = LIB, OBJ
    if profile:
        NVCC_FLAGS = NVCC_FLAGS + ["-DBOLT_PROFILE", "-DBOLT_XMODE"]
        lib, objdir = os.path.join(PKG, "libbolt_prof.so"), OBJ + "_prof"
    elif xmode:
        NVCC_FLAGS = NVCC_FLAGS + ["-DBOLT_XMODE"]
        lib, objdir = os.path.join(PKG, "libbolt_x.so"), OBJ + "_x"
    elif variant:
        # A/B variant: "name:-DFOO=1,-DBAR=2" -> libbolt_name.so (tools/ only)
        name, _, defs = variant.partition(":")
        NVCC_FLAGS = NVCC_FLAGS + [d for d in defs.split(",") if d]
        lib, objdir = os.path.join(PKG, f"libbolt_{name}.so"), OBJ + f"_{name}"
    os.makedirs(objdir, exist_ok=True)
    if not force and not _stale(lib, _deps()):
        return lib
    if force:
        for o in glob.glob(os.path.join(objdir, "*.o")):
            os.remove(o)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        results = list(ex.map(lambda s: _compile(s, verbose, objdir), _sources()))
    if verbose:
        for _, log in results:
            if log:
                sys.stderr.write(log)
    objs = [o for o, _ in results]
    tmp = lib + f".tmp{os.getpid()}"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    var = next((a.split("=", 1)[1] for a in sys.argv if a.startswith("--variant=")), "")
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv,
                profile="--profile" in sys.argv, xmode="--xmode" in sys.argv, variant=var))
