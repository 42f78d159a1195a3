"""In-tree build of the native libraries (no JIT cache, so the .so files travel
to the GPU box with the repo snapshot).

  libmoe_b200.so     sm_100a kernels + C ABI        (nvcc, -gencode sm_100a)
  libmoesim_b200.so  C++ drop-in of the reference moesim:: gating API, on top
                     of the C ABI                   (g++ -std=c++20)
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
HOST = os.path.join(HERE, "host")
INCLUDE = os.path.join(ROOT, "include")
EIGEN_MIN = os.path.join(ROOT, "third_party", "eigen_min")


def _json_dir() -> str:
    """nlohmann json 3.11 header shipped in the image (the reference's JSON
    dependency; used by the trace-file I/O)."""
    import sys
    for base in sys.path:
        d = os.path.join(base or ".", "include", "cudnn_frontend", "thirdparty", "nlohmann")
        if os.path.exists(os.path.join(d, "json.hpp")):
            return d
    raise RuntimeError("nlohmann json.hpp not found in the image")
LIB = os.path.join(HERE, "libmoe_b200.so")
LIBCXX = os.path.join(HERE, "libmoesim_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd, cwd=None):
    print("+", " ".join(cmd), flush=True)
    subprocess.run(cmd, check=True, cwd=cwd)


def build_cuda(force: bool = False, verbose_ptxas: bool = False) -> str:
    """Each .cu compiles to its own object (in parallel, only the stale ones),
    then one nvcc link into the shared library."""
    from concurrent.futures import ThreadPoolExecutor

    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    common = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + [
        os.path.join(INCLUDE, "moe_capi.h"), __file__]
    obj_dir = os.path.join(ROOT, "build", "obj")
    os.makedirs(obj_dir, exist_ok=True)
    objs = [os.path.join(obj_dir, os.path.basename(s)[:-3] + ".o") for s in srcs]
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", f"-I{INCLUDE}"]
    if verbose_ptxas:
        flags.insert(0, "-Xptxas=-v")
    todo = [(s, o) for s, o in zip(srcs, objs) if force or _stale(o, [s] + common)]

    def compile_one(so):
        s, o = so
        _run([NVCC, *flags, "-c", s, "-o", o])

    if todo:
        with ThreadPoolExecutor(max_workers=min(len(todo), os.cpu_count() or 4)) as ex:
            list(ex.map(compile_one, todo))
    if not force and not todo and not _stale(LIB, objs):
        return LIB
    _run([NVCC, *ARCH, "-shared", "-cudart", "static", "-o", LIB, *objs])
    return LIB


def build_cxx(force: bool = False) -> str:
    srcs = sorted(glob.glob(os.path.join(HOST, "*.cpp")))
    if not srcs:
        return ""
    deps = srcs + glob.glob(os.path.join(INCLUDE, "moesim", "*.hpp")) + [LIB, __file__]
    if not force and not _stale(LIBCXX, deps):
        return LIBCXX
    cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-Wall", "-Wextra", f"-I{INCLUDE}",
           f"-I{EIGEN_MIN}", f"-isystem{_json_dir()}", "-o", LIBCXX, *srcs, f"-L{HERE}", "-lmoe_b200",
           "-Wl,-rpath,$ORIGIN"]
    _run(cmd)
    return LIBCXX


TOOLS = os.path.join(ROOT, "tools")
BIN = os.path.join(ROOT, "build", "bin")


def build_tools(force: bool = False) -> None:
    """C++ host programs on the C++ API (no CUDA runtime linked directly)."""
    os.makedirs(BIN, exist_ok=True)
    for name in ("moesim_measure", "ep_p2p_demo"):
        src = os.path.join(TOOLS, name + ".cpp")
        exe = os.path.join(BIN, name)
        deps = [src, LIB, LIBCXX] + glob.glob(os.path.join(INCLUDE, "moesim", "*.hpp")) + [
            os.path.join(INCLUDE, "moe_capi.h")]
        if not force and not _stale(exe, deps):
            continue
        _run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", f"-I{INCLUDE}", f"-I{EIGEN_MIN}", "-o", exe,
              src, f"-L{HERE}", "-lmoesim_b200", "-lmoe_b200",
              "-Wl,-rpath,$ORIGIN/../../paper_2303_06182_b200"])


def build_all(force: bool = False) -> None:
    build_cuda(force)
    build_cxx(force)
    build_tools(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
