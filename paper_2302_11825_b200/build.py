"""Builds libbvc_b200.so in-tree: nvcc for sm_100a, no torch involved.

The library is the drop-in boundary: include/bvc_b200.h is its C ABI.
Objects compile in parallel; the shared library links CUDA's static runtime, so
it loads on a host without a GPU (every compute entry point then returns
BVC_ERR_NO_DEVICE — there is no CPU fallback).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_build")
LIB = os.path.join(OUT, "libbvc_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr", "-Xptxas", "-v"]
SOURCES = ["capi.cu", "capi_cache.cu", "capi_points.cu", "capi_splat.cu", "capi_walks.cu", "capi_stream.cu", "capi_comm.cu", "walk.cu", "walk3.cu", "gather.cu", "gather64.cu", "correct.cu", "probe.cu", "lbvh.cu", "sahbvh.cu", "host_scene.cpp", "io.cpp"]
HEADERS = ["capi_common.cuh", "tma.cuh", "device_math.cuh", "scene_dev.cuh", "scene3_dev.cuh", "internal.h", "gather.h", "host_scene.h"]


def _stale(obj: str, src: str) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "bvc_b200.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def _compile(src: str) -> tuple[str, str]:
    path = os.path.join(CSRC, src)
    obj = os.path.join(OUT, src + ".o")
    if not _stale(obj, path):
        return obj, ""
    cmd = [NVCC, *ARCH, *FLAGS, "-c", path, "-o", obj]
    if src.endswith(".cpp"):
        cmd = [NVCC, *ARCH, "-std=c++17", "-O3", "-Xcompiler", "-fPIC", "-c", path, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    os.makedirs(OUT, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(_compile, SOURCES))
    objs = [o for o, _ in results]
    if verbose:
        for _, log in results:
            if log:
                print(log, file=sys.stderr)
    if not os.path.exists(LIB) or any(os.path.getmtime(o) > os.path.getmtime(LIB) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-cudart", "static", "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
