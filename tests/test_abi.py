"""C-ABI checks that need no GPU: the library loads, exports every function
include/mpgabor.h declares, and validates dictionaries / computes layouts on the
host exactly as the paper's compatibility rules and reading Z3 say."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

from siggen import Dict, HANN, BLACKMAN, GAUSS, CONFIGS
from oracle import gabor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mpgabor.h")


@pytest.fixture(scope="module")
def mpg():
    from paper_2202_12380_b200.build import build_library
    build_library()
    import paper_2202_12380_b200.mpgabor as m
    return m


def _declared():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(mpgabor_\w+)\s*\(", txt, flags=re.M)))


def test_library_exports_every_declared_symbol(mpg):
    names = _declared()
    assert len(names) >= 10
    lib = ctypes.CDLL(mpg.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(mpg.EXPORTED), set(names) ^ set(mpg.EXPORTED)


def test_struct_layouts(mpg):
    assert ctypes.sizeof(mpg.mpg_dict) == 16
    assert mpg.ATOM_DTYPE.itemsize == 32            # mpg_atom
    assert ctypes.sizeof(mpg.mpg_result) == 48


@pytest.mark.parametrize("dicts,code", [
    ((Dict(HANN, 384, 96, 384), Dict(HANN, 512, 128, 512)), "EINVAL"),      # 384 not a power of two
    ((Dict(HANN, 256, 96, 256),), "EINCOMPAT"),                             # M/a not an integer
    ((Dict(HANN, 256, 64, 256), Dict(HANN, 512, 96, 512)), "EINCOMPAT"),    # 64 does not divide 96
    ((Dict(7, 256, 64, 256),), "EINVAL"),                                   # unknown window
    ((Dict(HANN, 0, 64, 256),), "EINVAL"),
    ((Dict(HANN, 256, 64, 32768),), "EINVAL"),                              # M > 16384
])
def test_create_rejects(mpg, dicts, code):
    with pytest.raises(mpg.MpgError) as e:
        mpg.mpgabor_create(dicts)
    assert code in str(e.value)
    assert mpg.mpgabor_last_error(None)


def test_create_accepts_and_layout_matches_oracle(mpg):
    for name in ("C0", "C1", "C2", "C3", "C4"):
        cfg = CONFIGS[name]
        h = mpg.mpgabor_create(cfg.dicts, mpg.MPG_F64)
        try:
            L, N, MR, off, rs = mpg.mpgabor_layout(h, cfg.Ls, len(cfg.dicts))
            lay = gabor.layout(cfg.dicts, cfg.Ls)
            assert L == lay.L and N == lay.N and MR == lay.MR and off[:-1] == lay.off and off[-1] == lay.P
            assert rs == lay.MR        # exchanged coefficient vectors are dense (row stride M_R)
        finally:
            mpg.mpgabor_destroy(h)


def test_precision_and_state_errors(mpg):
    with pytest.raises(mpg.MpgError):
        mpg.mpgabor_create([Dict(HANN, 16, 4, 16)], 7)
    h = mpg.mpgabor_create([Dict(HANN, 16, 4, 16)], mpg.MPG_F32)
    try:
        with pytest.raises(mpg.MpgError) as e:
            mpg.mpgabor_set_launch(h, 3, 0, 0, 0)
        assert "EINVAL" in str(e.value)
        with pytest.raises(mpg.MpgError):
            mpg.mpgabor_set_launch(h, 0, 0, 48, 0)
        mpg.mpgabor_set_launch(h, 4, 256, 32, 1)
        for bad in (-1, 9):
            with pytest.raises(mpg.MpgError) as e:
                mpg.mpgabor_set_batch(h, bad)
            assert "EINVAL" in str(e.value)
        for ok in (0, 1, 4, 8):
            mpg.mpgabor_set_batch(h, ok)
        for bad in (-1, 2):
            with pytest.raises(mpg.MpgError) as e:
                mpg.mpgabor_set_pedantic(h, bad)
            assert "EINVAL" in str(e.value)
        mpg.mpgabor_set_pedantic(h, 1)
        mpg.mpgabor_set_pedantic(h, 0)
        for bad in (256, 48, 24):
            with pytest.raises(mpg.MpgError):
                mpg.mpgabor_set_launch(h, bad, 0, 0, 0)
        for ok in (32, 64, 128):
            mpg.mpgabor_set_launch(h, ok, 0, 0, 0)   # grid mode of the one-selection loop
        dummy = ctypes.c_void_p(16)
        res = mpg.mpg_result()
        rc = mpg._lib.mpgabor_run_batch(h, dummy, 0, 1024, 10, -1.0, dummy, dummy, ctypes.byref(res), None)
        assert mpg.ERRORS[rc] == "EINVAL"
        rc = mpg._lib.mpgabor_run_reset(h, dummy, 1024, 10, -1.0, 0, dummy, dummy, ctypes.byref(res), None)
        assert mpg.ERRORS[rc] == "EINVAL"                 # reset_every < 1
        with pytest.raises(mpg.MpgError) as e:
            mpg.mpgabor_kernel_stats(h)             # before mpgabor_kernels
        assert "ESTATE" in str(e.value)
    finally:
        mpg.mpgabor_destroy(h)


def test_product_has_no_oracle_or_cpu_path():
    # the product package must not import the oracle nor contain a CPU fallback
    pkg = os.path.join(ROOT, "paper_2202_12380_b200")
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "import oracle" not in src and "from oracle" not in src, fn
            assert "numpy.fft" not in src and "np.fft" not in src, fn
