"""Build libmpgabor.so in-tree with nvcc for sm_100a (no JIT cache, no CPU fallback)."""
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libmpgabor.so")
SOURCES = ["csrc/analysis.cu", "csrc/mploop.cu", "csrc/mpmulti.cu", "csrc/synth.cu", "csrc/runtime.cu"]
HEADERS = ["csrc/common.cuh", "csrc/fft.cuh", "csrc/launch.h", "csrc/loopcore.cuh", "csrc/argmax.cuh", "../include/mpgabor.h"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-cudart", "static"]


def _stale():
    if not os.path.exists(LIB_PATH):
        return True
    t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(os.path.join(_HERE, s)) > t for s in SOURCES + HEADERS)


def build_library(force=False, verbose=False):
    if not force and not _stale():
        return LIB_PATH
    tmp = LIB_PATH + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, "-o", tmp, *SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.check_call(cmd, cwd=_HERE)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH
