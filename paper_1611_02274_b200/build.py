"""In-tree build of libbode.so (sm_100a) with nvcc.

    python -m paper_1611_02274_b200.build [--force]

Objects go to paper_1611_02274_b200/lib/obj, the shared library to
paper_1611_02274_b200/lib/libbode.so (git-ignored, shipped with the repo
snapshot to the GPU box). The CUDA runtime is linked statically, so the
library only needs the driver at run time.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
# BODE_BUILD_DIR / BODE_NVCC_EXTRA: an A/B variant of the library (e.g. lib/ab/<name>
# built with -D switches), loaded by the bench through BODE_LIB_PATH
LIB_DIR = os.environ.get("BODE_BUILD_DIR") or os.path.join(PKG, "lib")
OBJ_DIR = os.path.join(LIB_DIR, "obj")
SO = os.path.join(LIB_DIR, "libbode.so")
INCLUDE = os.path.join(os.path.dirname(PKG), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3",
         "-diag-suppress", "20012", "-I", INCLUDE] + os.environ.get("BODE_NVCC_EXTRA", "").split()


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _headers():
    return (glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h"))
            + glob.glob(os.path.join(INCLUDE, "*.h")) + glob.glob(os.path.join(INCLUDE, "*.cuh")))


def _stale(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _compile(src, verbose):
    obj = os.path.join(OBJ_DIR, os.path.basename(src) + ".o")
    if not _stale(obj, [src] + _headers()):
        return obj
    cmd = [NVCC, *ARCH, *FLAGS, "-Xptxas", "-v", "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    with open(obj + ".ptxas.txt", "w") as f:
        f.write(r.stderr)
    if verbose:
        print(f"[bode build] compiled {os.path.basename(src)}", flush=True)
    return obj


def build(force: bool = False, verbose: bool = True) -> str:
    os.makedirs(OBJ_DIR, exist_ok=True)
    if force:
        for f in glob.glob(os.path.join(OBJ_DIR, "*.o")):
            os.remove(f)
    srcs = _sources()
    with cf.ThreadPoolExecutor(max_workers=len(srcs)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    if _stale(SO, objs):
        cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", *objs, "-o", SO,
               "-Xlinker", "--no-undefined", "-lpthread"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stderr}")
        if verbose:
            print(f"[bode build] linked {SO}", flush=True)
    if not os.environ.get("BODE_BUILD_DIR"):
        build_examples(verbose)
    return SO


def build_examples(verbose: bool = True):
    """C++ drop-in example (examples/*.cpp) linked against libbode.so, and the
    out-of-tree problem libraries (examples/*.cu -> lib/lib<name>.so)."""
    repo = os.path.dirname(PKG)
    for src in glob.glob(os.path.join(repo, "examples", "*.cu")):
        so = os.path.join(LIB_DIR, "lib" + os.path.splitext(os.path.basename(src))[0] + ".so")
        if not _stale(so, [src, SO] + _headers() + [os.path.join(INCLUDE, "bode_problem.cuh")]):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-shared", "-Xptxas", "-v", src, "-L", LIB_DIR, "-lbode",
               "-Xlinker", f"-rpath,{LIB_DIR}", "-Xlinker", "-rpath,$ORIGIN", "-o", so]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"problem library build failed for {src}:\n{r.stderr}")
        with open(os.path.join(OBJ_DIR, os.path.basename(src) + ".ptxas.txt"), "w") as f:
            f.write(r.stderr)
        if verbose:
            print(f"[bode build] built {so}", flush=True)
    # test programs (tests/cpp): device problem libraries, then C++ tests linked
    # against libbode and those libraries
    test_libs = []
    for src in glob.glob(os.path.join(repo, "tests", "cpp", "*.cu")):
        name = os.path.splitext(os.path.basename(src))[0]
        so = os.path.join(LIB_DIR, "libtest_" + name + ".so")
        test_libs.append("test_" + name)
        if not _stale(so, [src, SO] + _headers() + [os.path.join(INCLUDE, "bode_problem.cuh")]):
            continue
        cmd = [NVCC, *ARCH, *FLAGS, "-shared", src, "-L", LIB_DIR, "-lbode",
               "-Xlinker", f"-rpath,{LIB_DIR}", "-Xlinker", "-rpath,$ORIGIN", "-o", so]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"test problem library build failed for {src}:\n{r.stderr}")
        if verbose:
            print(f"[bode build] built {so}", flush=True)
    for src in glob.glob(os.path.join(repo, "tests", "cpp", "*.cpp")):
        exe = os.path.join(LIB_DIR, os.path.splitext(os.path.basename(src))[0])
        libs = [os.path.join(LIB_DIR, "lib" + l + ".so") for l in test_libs]
        if not _stale(exe, [src, SO, os.path.join(INCLUDE, "bode.hpp")] + libs):
            continue
        cmd = ["g++", "-std=c++20", "-O2", "-Wall", "-I", INCLUDE, src, "-L", LIB_DIR,
               "-Wl,--no-as-needed", *[f"-l{l}" for l in test_libs], "-Wl,--as-needed",
               "-lbode", f"-Wl,-rpath,{LIB_DIR}", "-Wl,-rpath,$ORIGIN", "-o", exe]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"test program build failed for {src}:\n{r.stderr}")
        if verbose:
            print(f"[bode build] built {exe}", flush=True)
    for src in glob.glob(os.path.join(repo, "examples", "*.cpp")):
        exe = os.path.join(LIB_DIR, os.path.splitext(os.path.basename(src))[0])
        if not _stale(exe, [src, SO, os.path.join(INCLUDE, "bode.hpp")]):
            continue
        cmd = ["g++", "-std=c++20", "-O2", "-I", INCLUDE, src, "-L", LIB_DIR, "-lbode",
               f"-Wl,-rpath,{LIB_DIR}", "-Wl,-rpath,$ORIGIN", "-o", exe]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"example build failed for {src}:\n{r.stderr}")
        if verbose:
            print(f"[bode build] built {exe}", flush=True)


if __name__ == "__main__":
    build(force="--force" in sys.argv)
