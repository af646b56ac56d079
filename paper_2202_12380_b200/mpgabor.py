"""Thin ctypes binding of libmpgabor (include/mpgabor.h) -- argument marshalling only.

Functions carry the C names.  Device buffers are torch CUDA tensors; PyTorch is
used only for device memory and streams.  Every step of the method runs in the
CUDA kernels of libmpgabor.so; there is no CPU fallback: if the shared library
is missing this module raises at import time.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MPGABOR_LIB") or os.path.join(_HERE, "libmpgabor.so")  # override: A/B timing of builds

MPG_WIN_HANN, MPG_WIN_BLACKMAN, MPG_WIN_GAUSS = 1, 2, 3
MPG_F64, MPG_F32 = 0, 1
STOP_NAMES = {1: "maxit", 2: "errtol", 3: "negest", 4: "zero"}
ERRORS = {-1: "EINVAL", -2: "EINCOMPAT", -3: "ESTATE", -4: "ENOMEM", -5: "ECUDA", -6: "ELEN",
          -7: "ENONFINITE"}

ATOM_DTYPE = np.dtype([("w", "<i4"), ("m", "<i4"), ("n", "<i4"), ("flags", "<i4"),
                       ("re", "<f8"), ("im", "<f8")])


class mpg_dict(ctypes.Structure):
    _fields_ = [("win", ctypes.c_int32), ("gl", ctypes.c_int32), ("a", ctypes.c_int32),
                ("M", ctypes.c_int32)]


class mpg_result(ctypes.Structure):
    _fields_ = [("n_atoms", ctypes.c_int64), ("L_pad", ctypes.c_int64),
                ("stop_reason", ctypes.c_int32), ("cluster", ctypes.c_int32),
                ("E0", ctypes.c_double), ("E_final", ctypes.c_double), ("rounds", ctypes.c_int64)]


class MpgError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


if not os.path.exists(LIB_PATH):
    raise ImportError(f"libmpgabor.so not built ({LIB_PATH}); run __graft_entry__.build()")

_lib = ctypes.CDLL(LIB_PATH)
_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32

_SIGS = {
    "mpgabor_create": ([ctypes.POINTER(mpg_dict), _I32, _I32, ctypes.POINTER(_P)], ctypes.c_int),
    "mpgabor_kernels": ([_P, ctypes.c_double, _P], ctypes.c_int),
    "mpgabor_layout": ([_P, _I64, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64),
                        ctypes.POINTER(_I64), ctypes.POINTER(_I64)], ctypes.c_int),
    "mpgabor_run": ([_P, _P, _I64, _I64, ctypes.c_double, _P, _P, _P, ctypes.POINTER(mpg_result), _P],
                    ctypes.c_int),
    "mpgabor_synth": ([_P, _P, _I64, _P, _I64, _P], ctypes.c_int),
    "mpgabor_run_reset": ([_P, _P, _I64, _I64, ctypes.c_double, _I64, _P, _P, ctypes.POINTER(mpg_result), _P],
                          ctypes.c_int),
    "mpgabor_last_passes": ([_P, ctypes.POINTER(_I32)], ctypes.c_int),
    "mpgabor_run_batch": ([_P, _P, _I32, _I64, _I64, ctypes.c_double, _P, _P, ctypes.POINTER(mpg_result), _P],
                          ctypes.c_int),
    "mpgabor_decompose_host": ([_P, _P, _I64, _I64, ctypes.c_double, _P, _P, _P,
                                ctypes.POINTER(mpg_result), _P], ctypes.c_int),
    "mpgabor_set_launch": ([_P, _I32, _I32, _I32, _I32], ctypes.c_int),
    "mpgabor_set_batch": ([_P, _I32], ctypes.c_int),
    "mpgabor_set_pedantic": ([_P, _I32], ctypes.c_int),
    "mpgabor_launch_info": ([_P, ctypes.POINTER(_I32), ctypes.POINTER(_I32), ctypes.POINTER(_I32),
                             ctypes.POINTER(_I32), ctypes.POINTER(_I64)], ctypes.c_int),
    "mpgabor_kernel_stats": ([_P, ctypes.POINTER(_I64), ctypes.POINTER(_I64), ctypes.POINTER(_I64)],
                             ctypes.c_int),
    "mpgabor_kernel_box": ([_P, _I32, _I32, ctypes.POINTER(_I32), _P, ctypes.POINTER(ctypes.c_double)],
                           ctypes.c_int),
    "mpgabor_last_timing": ([_P, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double),
                             ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
    "mpgabor_residual": ([_P, _P, _P], ctypes.c_int),
    "mpgabor_launch_count": ([_P, ctypes.POINTER(_I64)], ctypes.c_int),
    "mpgabor_set_profile": ([_P, _I32], ctypes.c_int),
    "mpgabor_last_profile": ([_P, ctypes.POINTER(_I64)], ctypes.c_int),
    "mpgabor_destroy": ([_P], None),
    "mpgabor_last_error": ([_P], ctypes.c_char_p),
}
for _name, (_args, _res) in _SIGS.items():
    if os.environ.get("MPGABOR_LIB") and not hasattr(_lib, _name):
        continue  # A/B timing of an older build: calls it lacks are unavailable
    _f = getattr(_lib, _name)
    _f.argtypes = _args
    _f.restype = _res

EXPORTED = tuple(_SIGS)


def _check(h, rc):
    if rc != 0:
        raise MpgError(rc, _lib.mpgabor_last_error(h).decode())


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        import torch
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# ---------------------------------------------------------------------------
# C names
# ---------------------------------------------------------------------------
def mpgabor_create(dicts, precision=MPG_F64):
    """dicts: iterable of (win, gl, a, M) or objects with those attributes."""
    ds = []
    for d in dicts:
        if hasattr(d, "win"):
            ds.append(mpg_dict(int(d.win), int(d.gl), int(d.a), int(d.M)))
        else:
            ds.append(mpg_dict(*[int(v) for v in d]))
    arr = (mpg_dict * len(ds))(*ds)
    h = ctypes.c_void_p()
    rc = _lib.mpgabor_create(arr, len(ds), int(precision), ctypes.byref(h))
    if rc != 0:
        raise MpgError(rc, _lib.mpgabor_last_error(None).decode())
    return h


def mpgabor_kernels(h, thr, stream=None):
    _check(h, _lib.mpgabor_kernels(h, float(thr), _stream(stream)))


def mpgabor_layout(h, Ls, W):
    """(L_pad, N[W], M_R[W], coef_offset[W+1], row_stride[W])."""
    L = _I64()
    N = (_I64 * W)()
    MR = (_I64 * W)()
    rs = (_I64 * W)()
    off = (_I64 * (W + 1))()
    _check(h, _lib.mpgabor_layout(h, int(Ls), ctypes.byref(L), N, MR, rs, off))
    return L.value, list(N), list(MR), list(off), list(rs)


def mpgabor_run(h, x_dev, Ls, maxit, errdb, atoms_dev, energy_dev, coef_dev=None, stream=None):
    res = mpg_result()
    _check(h, _lib.mpgabor_run(h, _ptr(x_dev), int(Ls), int(maxit), float(errdb), _ptr(atoms_dev),
                               _ptr(energy_dev), _ptr(coef_dev), ctypes.byref(res), _stream(stream)))
    return res


def mpgabor_run_reset(h, x_dev, Ls, maxit, errdb, reset_every, atoms_dev, energy_dev, stream=None):
    res = mpg_result()
    _check(h, _lib.mpgabor_run_reset(h, _ptr(x_dev), int(Ls), int(maxit), float(errdb), int(reset_every),
                                     _ptr(atoms_dev), _ptr(energy_dev), ctypes.byref(res), _stream(stream)))
    return res


def mpgabor_run_batch(h, x_dev, B, Ls, maxit, errdb, atoms_dev, energy_dev, stream=None):
    res = (mpg_result * int(B))()
    _check(h, _lib.mpgabor_run_batch(h, _ptr(x_dev), int(B), int(Ls), int(maxit), float(errdb), _ptr(atoms_dev),
                                     _ptr(energy_dev), res, _stream(stream)))
    return list(res)


def mpgabor_last_passes(h):
    n = _I32()
    _check(h, _lib.mpgabor_last_passes(h, ctypes.byref(n)))
    return n.value


def mpgabor_synth(h, atoms_dev, n_atoms, y_dev, Ls, stream=None):
    _check(h, _lib.mpgabor_synth(h, _ptr(atoms_dev), int(n_atoms), _ptr(y_dev), int(Ls), _stream(stream)))


def mpgabor_decompose_host(h, x_host, maxit, errdb, atoms_host=None, energy_host=None, y_host=None,
                           stream=None):
    """x_host, atoms_host, energy_host, y_host: numpy arrays (pinned torch CPU tensors also work)."""
    res = mpg_result()

    def hp(a):
        if a is None:
            return None
        if hasattr(a, "data_ptr"):
            return ctypes.c_void_p(a.data_ptr())
        return ctypes.c_void_p(a.ctypes.data)

    _check(h, _lib.mpgabor_decompose_host(h, hp(x_host), int(x_host.shape[0]), int(maxit), float(errdb),
                                          hp(atoms_host), hp(energy_host), hp(y_host), ctypes.byref(res),
                                          _stream(stream)))
    return res


def mpgabor_set_launch(h, cluster=0, threads=0, tile_width=0, records=0):
    _check(h, _lib.mpgabor_set_launch(h, int(cluster), int(threads), int(tile_width), int(records)))


def mpgabor_set_batch(h, max_batch):
    _check(h, _lib.mpgabor_set_batch(h, int(max_batch)))


def mpgabor_set_pedantic(h, on):
    _check(h, _lib.mpgabor_set_pedantic(h, int(on)))


def mpgabor_launch_info(h):
    c, t, tw, r = _I32(), _I32(), _I32(), _I32()
    sm = _I64()
    _check(h, _lib.mpgabor_launch_info(h, ctypes.byref(c), ctypes.byref(t), ctypes.byref(tw), ctypes.byref(r),
                                       ctypes.byref(sm)))
    return {"cluster": c.value, "threads": t.value, "tile_width": tw.value,
            "records": "shared" if r.value == 1 else "global", "smem_bytes": sm.value}


def mpgabor_kernel_stats(h):
    a, b, c = _I64(), _I64(), _I64()
    _check(h, _lib.mpgabor_kernel_stats(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def mpgabor_kernel_box(h, u, v):
    box = (_I32 * 4)()
    mx = ctypes.c_double()
    _check(h, _lib.mpgabor_kernel_box(h, int(u), int(v), box, None, ctypes.byref(mx)))
    mu_lo, mu_hi, nu_lo, nu_hi = list(box)
    vals = np.zeros((nu_hi - nu_lo + 1, mu_hi - mu_lo + 1), dtype=np.complex128)
    _check(h, _lib.mpgabor_kernel_box(h, int(u), int(v), box, ctypes.c_void_p(vals.ctypes.data),
                                      ctypes.byref(mx)))
    return (mu_lo, mu_hi, nu_lo, nu_hi), vals, mx.value


def mpgabor_last_timing(h):
    a, b, c = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    _check(h, _lib.mpgabor_last_timing(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
    return a.value, b.value, c.value


def mpgabor_residual(h, out_dev, stream=None):
    _check(h, _lib.mpgabor_residual(h, _ptr(out_dev), _stream(stream)))


def mpgabor_launch_count(h):
    n = _I64()
    _check(h, _lib.mpgabor_launch_count(h, ctypes.byref(n)))
    return n.value


def mpgabor_set_profile(h, mode):
    _check(h, _lib.mpgabor_set_profile(h, int(mode)))


def mpgabor_last_profile(h):
    c = (_I64 * 512)()
    _check(h, _lib.mpgabor_last_profile(h, c))
    return list(c)


def mpgabor_destroy(h):
    _lib.mpgabor_destroy(h)


def mpgabor_last_error(h=None):
    return _lib.mpgabor_last_error(h).decode()


# ---------------------------------------------------------------------------
# convenience object (still marshalling only)
# ---------------------------------------------------------------------------
@dataclass
class RunOutput:
    atoms: np.ndarray      # ATOM_DTYPE[n]
    energy: np.ndarray     # E_0 .. E_n
    stop: int
    E0: float
    L_pad: int
    cluster: int
    coef: object = None    # torch complex128 [P_R] on device (or None)
    atoms_dev: object = None
    rounds: int = 0        # persistent-loop rounds (multi-selection)

    @property
    def n(self):
        return self.atoms.size

    @property
    def stop_name(self):
        return STOP_NAMES.get(self.stop, "?")

    def index(self, offsets, MR):
        off = np.asarray(offsets)
        mr = np.asarray(MR)
        return off[self.atoms["w"]] + self.atoms["n"].astype(np.int64) * mr[self.atoms["w"]] + self.atoms["m"]


class MPGabor:
    """Handle wrapper: MPGabor(dicts, thr, precision).run(x) -> RunOutput."""

    def __init__(self, dicts, thr=1e-4, precision="f64", stream=None):
        import torch
        self.torch = torch
        self.dicts = tuple(dicts)
        self.W = len(self.dicts)
        self.precision = MPG_F64 if precision in ("f64", MPG_F64) else MPG_F32
        self.h = mpgabor_create(self.dicts, self.precision)
        self.thr = float(thr)
        mpgabor_kernels(self.h, self.thr, stream)

    def close(self):
        if self.h is not None:
            mpgabor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def layout(self, Ls):
        return mpgabor_layout(self.h, Ls, self.W)

    def set_launch(self, cluster=0, threads=0, tile_width=0, records=0):
        mpgabor_set_launch(self.h, cluster, threads, tile_width, records)

    def launch_info(self):
        return mpgabor_launch_info(self.h)

    def set_batch(self, max_batch):
        mpgabor_set_batch(self.h, max_batch)

    def set_pedantic(self, on):
        mpgabor_set_pedantic(self.h, on)

    def alloc(self, maxit, Ls, want_coef=False):
        torch = self.torch
        atoms = torch.empty(max(int(maxit), 1) * ATOM_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        energy = torch.empty(int(maxit) + 1, dtype=torch.float64, device="cuda")
        coef = None
        if want_coef:
            P = self.layout(Ls)[3][-1]
            coef = torch.empty(2 * P, dtype=torch.float64, device="cuda")
        return atoms, energy, coef

    def run(self, x, maxit, errdb=-math.inf, want_coef=False, bufs=None, stream=None, fetch=True):
        torch = self.torch
        if not isinstance(x, torch.Tensor):
            x = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).cuda()
        assert x.dtype == torch.float64 and x.is_cuda and x.is_contiguous()
        Ls = x.shape[0]
        atoms, energy, coef = bufs if bufs is not None else self.alloc(maxit, Ls, want_coef)
        res = mpgabor_run(self.h, x, Ls, maxit, errdb, atoms, energy, coef, stream)
        if not fetch:
            return res, (atoms, energy, coef)
        n = res.n_atoms
        at = np.frombuffer(atoms[: n * ATOM_DTYPE.itemsize].cpu().numpy().tobytes(), dtype=ATOM_DTYPE)
        en = energy[: n + 1].cpu().numpy()
        return RunOutput(at, en, res.stop_reason, res.E0, res.L_pad, res.cluster,
                         coef.view(torch.complex128) if coef is not None else None, atoms, res.rounds)

    def run_reset(self, x, maxit, errdb=-math.inf, reset_every=1000, stream=None):
        """Alg. 2 (resets); returns RunOutput (passes in .rounds is the loop rounds)."""
        torch = self.torch
        if not isinstance(x, torch.Tensor):
            x = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)).cuda()
        assert x.dtype == torch.float64 and x.is_cuda and x.is_contiguous()
        Ls = x.shape[0]
        atoms, energy, _ = self.alloc(maxit, Ls)
        res = mpgabor_run_reset(self.h, x, Ls, maxit, errdb, reset_every, atoms, energy, stream)
        n = res.n_atoms
        at = np.frombuffer(atoms[: n * ATOM_DTYPE.itemsize].cpu().numpy().tobytes(), dtype=ATOM_DTYPE)
        en = energy[: n + 1].cpu().numpy()
        return RunOutput(at, en, res.stop_reason, res.E0, res.L_pad, res.cluster, None, atoms, res.rounds)

    def run_batch(self, X, maxit, errdb=-math.inf, stream=None, fetch=True):
        """B independent signals X[B][Ls] (one cluster each); returns a list of RunOutput
        (fetch=False: the list of mpg_result and the device atom / energy buffers)."""
        torch = self.torch
        if not isinstance(X, torch.Tensor):
            X = torch.as_tensor(np.ascontiguousarray(X, dtype=np.float64)).cuda()
        assert X.dtype == torch.float64 and X.is_cuda and X.is_contiguous() and X.dim() == 2
        B, Ls = X.shape
        atoms = torch.empty(B * max(int(maxit), 1) * ATOM_DTYPE.itemsize, dtype=torch.uint8, device="cuda")
        energy = torch.empty(B * (int(maxit) + 1), dtype=torch.float64, device="cuda")
        res = mpgabor_run_batch(self.h, X, B, Ls, maxit, errdb, atoms, energy, stream)
        if not fetch:
            return res, atoms, energy
        ab = atoms.cpu().numpy().tobytes()
        en = energy.cpu().numpy()
        outs = []
        for b, r in enumerate(res):
            n = r.n_atoms
            a0 = b * int(maxit) * ATOM_DTYPE.itemsize
            at = np.frombuffer(ab[a0: a0 + n * ATOM_DTYPE.itemsize], dtype=ATOM_DTYPE)
            e0 = b * (int(maxit) + 1)
            outs.append(RunOutput(at, en[e0: e0 + n + 1].copy(), r.stop_reason, r.E0, r.L_pad, r.cluster,
                                  None, None, r.rounds))
        return outs

    def last_passes(self):
        return mpgabor_last_passes(self.h)

    def synth(self, atoms_dev, n_atoms, Ls, stream=None):
        torch = self.torch
        y = torch.empty(int(Ls), dtype=torch.float64, device="cuda")
        mpgabor_synth(self.h, atoms_dev, n_atoms, y, Ls, stream)
        return y

    def kernel_stats(self):
        return mpgabor_kernel_stats(self.h)

    def kernel_box(self, u, v):
        return mpgabor_kernel_box(self.h, u, v)

    def residual(self, Ls, stream=None):
        """Residual c^ of the last run as a complex128 torch tensor [P_R] on the device."""
        torch = self.torch
        P = self.layout(Ls)[3][-1]
        out = torch.empty(2 * P, dtype=torch.float64, device="cuda")
        mpgabor_residual(self.h, out, stream)
        return out.view(torch.complex128)

    def launch_count(self):
        return mpgabor_launch_count(self.h)

    def set_profile(self, mode):
        mpgabor_set_profile(self.h, mode)

    def last_profile(self):
        return mpgabor_last_profile(self.h)

    def last_timing(self):
        return mpgabor_last_timing(self.h)
