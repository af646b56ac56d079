"""ctypes wrapper of oracle/mploop.c (TEST INFRASTRUCTURE ONLY).

``mp_run(setup, maxit, errdb)`` runs the coefficient-domain MP loop of
SURVEY.md §8(c) O7 on a copy of the setup's residual grids and returns the
atom list, the energy-estimate trace E_k, the top-2 gaps and the final
residual / solution grids.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mploop.c")
_LIB = os.path.join(_HERE, "libmploop.so")

ATOM_DTYPE = np.dtype([("w", "<i4"), ("m", "<i4"), ("n", "<i4"), ("flags", "<i4"),
                       ("re", "<f8"), ("im", "<f8")])

STOP_NAMES = {1: "maxit", 2: "errtol", 3: "negest", 4: "zero"}


class _Dict(ctypes.Structure):
    _fields_ = [("a", ctypes.c_int32), ("M", ctypes.c_int32), ("N", ctypes.c_int32),
                ("MR", ctypes.c_int32), ("off", ctypes.c_int64)]


class _Kern(ctypes.Structure):
    _fields_ = [("a_c", ctypes.c_int32), ("M_c", ctypes.c_int32),
                ("mu_lo", ctypes.c_int32), ("mu_hi", ctypes.c_int32),
                ("nu_lo", ctypes.c_int32), ("nu_hi", ctypes.c_int32),
                ("h", ctypes.c_void_p)]


def build(force: bool = False) -> str:
    """Compile mploop.c with gcc (no FMA contraction, single thread)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-D_GNU_SOURCE", "-ffp-contract=off",
                               "-fno-fast-math", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        _lib.orc_mp_run.restype = ctypes.c_int
        _lib.orc_mp_run.argtypes = [
            ctypes.c_int32, ctypes.POINTER(_Dict), ctypes.POINTER(_Kern), ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int32)]
    return _lib


@dataclass
class MpResult:
    atoms: np.ndarray        # ATOM_DTYPE[n]
    energy: np.ndarray       # E_0 .. E_n
    gaps: np.ndarray         # (s1 - s2)/s1 at each selection
    stop: int
    res: np.ndarray          # final residual, all dictionaries concatenated (complex128[P])
    sol: np.ndarray          # solution grid (complex128[P])
    index: np.ndarray        # global index p of each selected atom

    @property
    def n(self):
        return self.atoms.size

    @property
    def stop_name(self):
        return STOP_NAMES.get(self.stop, "?")


def error_tolerance(errdb: float, E0: float) -> float:
    """Absolute stop level 10^(errdb/10) E_0; -inf disables it."""
    if errdb == -math.inf:
        return -math.inf
    return 10.0 ** (errdb / 10.0) * E0


def mp_run(setup, maxit: int, errdb: float = -math.inf, full_scan: bool = False,
           want_gaps: bool = True, etol: float | None = None, pedantic: bool = False) -> MpResult:
    """Alg. 1 on the setup's grids; ``etol`` (absolute energy level) overrides errdb;
    ``pedantic`` selects by the Eq. (20) energy instead of |c^|^2."""
    lib = _load()
    lay = setup.lay
    W = len(setup.dicts)
    dd = (_Dict * W)(*[_Dict(d.a, d.M, lay.N[w], lay.MR[w], lay.off[w])
                       for w, d in enumerate(setup.dicts)])
    hs = [np.ascontiguousarray(K.h, dtype=np.complex128) for K in setup.K]
    kk = (_Kern * (W * W))(*[_Kern(K.a_c, K.M_c, K.mu_lo, K.mu_hi, K.nu_lo, K.nu_hi,
                                   h.ctypes.data) for K, h in zip(setup.K, hs)])
    res = np.concatenate([g.ravel() for g in setup.grids]).astype(np.complex128)
    sol = np.zeros_like(res)
    maxit = int(maxit)
    atoms = np.zeros(max(maxit, 1), dtype=ATOM_DTYPE)
    energy = np.zeros(maxit + 1)
    gaps = np.zeros(max(maxit, 1))
    n_done = ctypes.c_int64(0)
    stop = ctypes.c_int32(0)
    rc = lib.orc_mp_run(W, dd, kk, res.ctypes.data, sol.ctypes.data, maxit,
                        error_tolerance(errdb, setup.E0) if etol is None else etol, setup.E0, int(full_scan),
                        int(pedantic),
                        atoms.ctypes.data, energy.ctypes.data,
                        gaps.ctypes.data if want_gaps else None,
                        ctypes.byref(n_done), ctypes.byref(stop))
    if rc != 0:
        raise RuntimeError(f"orc_mp_run failed: {rc}")
    n = n_done.value
    at = atoms[:n].copy()
    off = np.asarray(lay.off)
    MR = np.asarray(lay.MR)
    index = off[at["w"]] + at["n"].astype(np.int64) * MR[at["w"]] + at["m"]
    return MpResult(at, energy[: n + 1].copy(), gaps[:n].copy() if want_gaps else None,
                    stop.value, res, sol, index)


@dataclass
class ResetResult:
    atoms: np.ndarray        # ATOM_DTYPE[n], all passes in order
    energy: np.ndarray       # E_0 .. E_n: the true residual energy at every pass start, estimates inside
    stop: int
    passes: int
    residual: np.ndarray     # final signal-domain residual r_out (length L)
    index: np.ndarray

    @property
    def n(self):
        return self.atoms.size

    @property
    def stop_name(self):
        return STOP_NAMES.get(self.stop, "?")


def mp_run_reset(x, dicts, thr, maxit: int, errdb: float, reset_every: int, K=None) -> ResetResult:
    """Approximate coefficient-domain MP with reset, Alg. 2.

    Outer loop: while the stopping criterion (maxit atoms; true residual energy
    E_out <= 10^(errdb/10) ||x||^2) is not met, run Alg. 1 from
    c^ = D^* r_out with E_k starting at E_out (step 1), until the reset criterion:
    ``reset_every`` selections, or the inner estimate reaching the stop level or a
    negative estimate; a zero largest score ends the run.  Then
    c_out += c, r_out -= D c (synthesis, Eq. (18)) and E_out = ||r_out||^2 (step 2).
    The problem lives on the zero-padded signal (reading Z3): r_out has length L.
    """
    from . import gabor
    dicts = tuple(dicts)
    Ls = x.size
    lay = gabor.layout(dicts, Ls)
    L = lay.L
    if K is None:
        K = gabor.kernels(dicts, thr)
    r = np.zeros(L)
    r[:Ls] = x
    E0 = float(np.dot(x, x))
    etol = error_tolerance(errdb, E0)
    atoms, energy = [], [E0]
    k, passes, stop = 0, 0, 1
    while True:
        if k >= maxit:
            stop = 1
            break
        S = gabor.Setup.build(r, dicts, thr, K)          # c^ = D^* r_out, E_k = E_out = ||r_out||^2
        energy[-1] = S.E0
        inner = mp_run(S, min(int(reset_every), maxit - k), etol=etol, want_gaps=False)
        passes += 1
        if inner.n == 0:
            stop = inner.stop                             # errtol on E_out, or zero score
            break
        atoms.append(inner.atoms)
        energy.extend(inner.energy[1:].tolist())
        r = r - gabor.synthesize(inner.atoms, dicts, L, L)   # r_out -= D c
        k += inner.n
        if inner.stop == 4:
            stop = 4
            break
    at = np.concatenate(atoms) if atoms else np.zeros(0, dtype=ATOM_DTYPE)
    off = np.asarray(lay.off)
    MR = np.asarray(lay.MR)
    index = off[at["w"]] + at["n"].astype(np.int64) * MR[at["w"]] + at["m"]
    return ResetResult(at, np.asarray(energy), stop, passes, r, index)
