"""Build libmpgabor.so in-tree with nvcc for sm_100a (no JIT cache, no CPU fallback).

Every translation unit is compiled to an object in parallel (build/ next to csrc/),
then linked into one shared library with the CUDA runtime linked statically."""
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpgabor.so")
SOURCES = ["csrc/analysis.cu", "csrc/mploop.cu", "csrc/mpmulti.cu", "csrc/synth.cu", "csrc/runtime.cu"]
HEADERS = ["csrc/common.cuh", "csrc/fft.cuh", "csrc/launch.h", "csrc/loopcore.cuh", "csrc/argmax.cuh", "../include/mpgabor.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]
LDFLAGS = ARCH + ["-shared", "-cudart", "static"]


def _stale():
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(os.path.join(_HERE, s)) > t for s in SOURCES + HEADERS)


def build_library(force=False, verbose=False):
    if not force and not _stale():
        return LIB_PATH
    objdir = os.path.join(_HERE, "build")
    os.makedirs(objdir, exist_ok=True)
    tag = f".{os.getpid()}.o"

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + tag)
        cmd = [NVCC, *CFLAGS, "-c", "-o", obj, src]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd, cwd=_HERE)
        return obj

    with ThreadPoolExecutor(len(SOURCES)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    try:
        subprocess.check_call([NVCC, *LDFLAGS, "-o", tmp, *objs], cwd=_HERE)
        os.replace(tmp, LIB_PATH)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return LIB_PATH
