"""Build libmpgabor.so in-tree with nvcc for sm_100a (no JIT cache, no CPU fallback).

Every translation unit is compiled to an object in parallel (build/ next to csrc/),
then linked into one shared library with the CUDA runtime linked statically."""
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpgabor.so")
SOURCES = ["csrc/mpmulti_f64_cluster.cu", "csrc/mpmulti_f64_grid.cu", "csrc/mpmulti_f32_cluster.cu",
           "csrc/mpmulti_f32_grid.cu", "csrc/mploop.cu", "csrc/analysis.cu", "csrc/mpmulti.cu", "csrc/synth.cu",
           "csrc/runtime.cu"]
HEADERS = ["csrc/common.cuh", "csrc/fft.cuh", "csrc/launch.h", "csrc/loopcore.cuh", "csrc/argmax.cuh",
           "csrc/mpmulti.cuh", "../include/mpgabor.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
LDFLAGS = ARCH + ["-shared", "-cudart", "static"]


def _stale():
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(os.path.join(_HERE, s)) > t for s in SOURCES + HEADERS)


def build_library(force=False, verbose=False, extra=(), out=None):
    """Compile and link; `extra` nvcc flags and another output path build A/B variants."""
    target = out or LIB_PATH
    if not force and not extra and out is None and not _stale():
        return LIB_PATH
    objdir = os.path.join(_HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    tag = f".{os.getpid()}.o"

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + tag)
        cmd = [NVCC, *CFLAGS, *extra, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd, cwd=_HERE)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = target + f".tmp{os.getpid()}"
    try:
        subprocess.check_call([NVCC, *LDFLAGS, "-o", tmp, *objs], cwd=_HERE)
        os.replace(tmp, target)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return target
