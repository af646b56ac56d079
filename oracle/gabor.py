"""Oracle: windows, DGT, Gram (cross-)kernels, synthesis -- numpy, fp64.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Plain, slow, obviously
correct; numpy's FFT is used as a library primitive (one DFT per frame / per
time lag) exactly where the definition is a DFT.

Citations ``P:<line>`` refer to /root/reference/PAPER.md; readings Z1..Z22 are
SURVEY.md §8(c) and are restated in DESIGN.md §2.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

HANN, BLACKMAN, GAUSS = 1, 2, 3


# ---------------------------------------------------------------------------
# O2 windows ("g in R^L, ||g||_2 = 1"; Fig. 1 P:591-605 names Gauss,
# Hann, Blackman; reading Z1: periodic, zero-phase, offsets -floor(gl/2) ..
# ceil(gl/2)-1; Z2: Gauss tfr = a*M)
# ---------------------------------------------------------------------------
def window(d):
    """Return (j0, g): g[i] is the unit-norm window at signed offset j0 + i."""
    gl = int(d.gl)
    if gl < 1:
        raise ValueError("gl must be >= 1")
    j = np.arange(-(gl // 2), gl - gl // 2, dtype=np.float64)
    if d.win == HANN:
        g = 0.5 + 0.5 * np.cos(2.0 * np.pi * j / gl)
    elif d.win == BLACKMAN:
        g = 0.42 + 0.5 * np.cos(2.0 * np.pi * j / gl) + 0.08 * np.cos(4.0 * np.pi * j / gl)
    elif d.win == GAUSS:
        g = np.exp(-np.pi * j * j / (float(d.a) * float(d.M)))
    else:
        raise ValueError(f"unknown window kind {d.win}")
    g = g / np.sqrt(np.sum(g * g))
    return -(gl // 2), g


# ---------------------------------------------------------------------------
# O1 validation and padding (P:287-306 compatibility; reading Z3: zero-pad Ls
# to a multiple of lcm{a_w, M_w})
# ---------------------------------------------------------------------------
@dataclass
class Layout:
    L: int
    N: list
    MR: list
    off: list          # coefficient offset of dictionary w in the global index p
    P: int             # total reduced coefficients


def validate(dicts):
    for d in dicts:
        if d.gl < 1 or d.a < 1 or d.M < 1:
            raise ValueError("gl, a, M must be >= 1")
        if d.M % d.a:
            raise ValueError("M/a must be a positive integer (P:300-301)")
    for u in dicts:
        for v in dicts:
            if max(u.a, v.a) % min(u.a, v.a) or max(u.M, v.M) % min(u.M, v.M):
                raise ValueError("incompatible pair (P:296-300)")


def layout(dicts, Ls):
    validate(dicts)
    ell = 1
    for d in dicts:
        ell = math.lcm(ell, d.a, d.M)
    L = -(-Ls // ell) * ell
    N = [L // d.a for d in dicts]
    MR = [d.M // 2 + 1 for d in dicts]
    off, p = [], 0
    for n, m in zip(N, MR):
        off.append(p)
        p += n * m
    return Layout(L, N, MR, off, p)


# ---------------------------------------------------------------------------
# O3 DGT: c(m,n) = <x, d_{m,n}> = sum_j x(na+j) g(j) e^{-i 2 pi m j / M}
# (Eq. (3), time-invariant phase; analysis P:913-921; reduced bins
# m = 0..floor(M/2) P:847-849)
# ---------------------------------------------------------------------------
def dgt(x, d):
    L = x.size
    j0, g = window(d)
    N = L // d.a
    j = j0 + np.arange(g.size)
    out = np.empty((N, d.M // 2 + 1), dtype=np.complex128)
    step = max(1, (1 << 22) // max(d.M, g.size))
    for n0 in range(0, N, step):
        n = np.arange(n0, min(N, n0 + step))
        fr = x[(n[:, None] * d.a + j[None, :]) % L] * g[None, :]
        b = np.zeros((n.size, d.M))
        for c0 in range(0, g.size, d.M):           # fold j mod M (gl may exceed M)
            cols = np.arange(c0, min(g.size, c0 + d.M))
            b[:, (j[cols]) % d.M] += fr[:, cols]
        out[n] = np.fft.fft(b, axis=1)[:, : d.M // 2 + 1]
    return out


def analysis_all(x, dicts, lay):
    xp = np.zeros(lay.L)
    xp[: x.size] = x
    return [dgt(xp, d) for d in dicts]


# ---------------------------------------------------------------------------
# O4 (cross-)kernels on the common grid (Eqs. (14)-(15) P:549-561, single
# dictionary P:575-595, cross-kernels Eq. (17), App. A1-A2 of
# SURVEY.md):
#   h_{u,v}(mu,nu) = sum_s g_u(s + nu a_c) g_v(s) e^{-i 2 pi mu s / M_c}
# with a_c = min(a_u,a_v), M_c = max(M_u,M_v), mu signed in (-M_c/2, M_c/2],
# nu over every lag with window overlap (reading Z8).  Threshold Eq. (7)
# P:407-413 applied relative to the kernel's own max|h| (Z5), strict (Z6),
# sub-threshold entries zeroed inside the bounding box (Z7).
# ---------------------------------------------------------------------------
@dataclass
class Kernel:
    a_c: int
    M_c: int
    mu_lo: int
    mu_hi: int
    nu_lo: int
    nu_hi: int
    h: np.ndarray            # [nu_hi-nu_lo+1, mu_hi-mu_lo+1] complex128, zeros where dropped
    mx: float                # max |h| before truncation
    kept: int                # number of entries with |h| > thr*mx


def kernel_full(du, dv):
    """Untruncated h_{u,v}: returns (a_c, M_c, nu_lo, H) with H[i, mu mod M_c] at nu = nu_lo+i."""
    a_c, M_c = min(du.a, dv.a), max(du.M, dv.M)
    ju0, gu = window(du)
    jv0, gv = window(dv)
    ju1, jv1 = ju0 + gu.size - 1, jv0 + gv.size - 1
    nu_lo = -((jv1 - ju0) // a_c)                      # ceil((ju0 - jv1)/a_c)
    nu_hi = (ju1 - jv0) // a_c
    B = np.zeros((nu_hi - nu_lo + 1, M_c))
    for i, nu in enumerate(range(nu_lo, nu_hi + 1)):
        s = np.arange(max(jv0, ju0 - nu * a_c), min(jv1, ju1 - nu * a_c) + 1)
        if s.size:
            np.add.at(B[i], s % M_c, gu[s + nu * a_c - ju0] * gv[s - jv0])
    return a_c, M_c, nu_lo, np.fft.fft(B, axis=1)


def cross_kernel(du, dv, thr):
    if not (0.0 <= thr < 1.0):
        raise ValueError("threshold must be in [0, 1)")
    a_c, M_c, nu0, H = kernel_full(du, dv)
    mag = np.abs(H)
    mx = float(mag.max())
    keep = mag > thr * mx
    nus, mus = np.nonzero(keep)
    mus_signed = np.where(2 * mus <= M_c, mus, mus - M_c)
    mu_lo, mu_hi = int(mus_signed.min()), int(mus_signed.max())
    nu_lo, nu_hi = int(nus.min()) + nu0, int(nus.max()) + nu0
    rows = np.arange(nu_lo - nu0, nu_hi - nu0 + 1)
    cols = np.arange(mu_lo, mu_hi + 1) % M_c
    h = np.where(keep[np.ix_(rows, cols)], H[np.ix_(rows, cols)], 0.0)
    return Kernel(a_c, M_c, mu_lo, mu_hi, nu_lo, nu_hi, np.ascontiguousarray(h), mx,
                  int(keep.sum()))


def kernels(dicts, thr):
    """K[u*W + v] = h_{u,v}: kernel used when an atom of u is selected and v is updated."""
    return [cross_kernel(du, dv, thr) for du in dicts for dv in dicts]


def kernel_value(K, mu, nu):
    """h(mu, nu) of a truncated kernel (0 outside the box); mu is reduced to signed range."""
    mu = mu % K.M_c
    if 2 * mu > K.M_c:
        mu -= K.M_c
    if K.mu_lo <= mu <= K.mu_hi and K.nu_lo <= nu <= K.nu_hi:
        return complex(K.h[nu - K.nu_lo, mu - K.mu_lo])
    return 0j


# ---------------------------------------------------------------------------
# O8 synthesis, Eq. (18): x = sum_w D_w c_w + conj(D_w) conj(c_w),
# conj term zeroed for m = 0 and m = M/2.  Atom by atom.
# ---------------------------------------------------------------------------
def synthesize(atoms, dicts, L, Ls=None):
    """atoms: structured array/dict with fields w, m, n, flags, re, im."""
    y = np.zeros(L)
    w_all = np.asarray(atoms["w"])
    for w, d in enumerate(dicts):
        sel = np.nonzero(w_all == w)[0]
        if sel.size == 0:
            continue
        j0, g = window(d)
        j = j0 + np.arange(g.size)
        m = np.asarray(atoms["m"])[sel]
        n = np.asarray(atoms["n"])[sel]
        c = np.asarray(atoms["re"])[sel] + 1j * np.asarray(atoms["im"])[sel]
        selfc = (m == 0) | (2 * m == d.M)
        mult = np.where(selfc, 1.0, 2.0)
        step = max(1, (1 << 22) // g.size)
        for k0 in range(0, sel.size, step):
            k = slice(k0, k0 + step)
            ph = np.exp(2j * np.pi * np.outer(m[k], j) / d.M)
            contrib = (mult[k, None] * np.real(c[k, None] * ph)) * g[None, :]
            pos = (n[k, None] * d.a + j[None, :]) % L
            y += np.bincount(pos.ravel(), weights=contrib.ravel(), minlength=L)
    return y if Ls is None else y[:Ls]


# ---------------------------------------------------------------------------
# Residual at single coefficients, one by one: c^_K(p) = c^_0(p) - sum_k (update
# of atom k at p).  The update of atom k = (u, k, j, c~) at target p = (v, m, n) is
# Alg. 3 restricted to one target: with a_c, M_c of the pair, the
# time lag nu = (n a_v - j a_u)/a_c (circular, signed) and the modulation
# omega_R^{(k' nu) mod R} (Eq. (15)),
#   direct:   - c~ omega h(m s_m - k', nu)
#   conj:     - conj(c~ omega h(((M_v - m) mod M_v) s_m - k', nu))   (pair atoms, Z14)
# (mu reduced to the signed range, h = 0 outside the kept box).
# ---------------------------------------------------------------------------
def residual_at(setup, atoms, points):
    """points: int array of global indices p; returns complex128 c^_K(p)."""
    lay, dicts, W = setup.lay, setup.dicts, len(setup.dicts)
    L = lay.L
    res0 = np.concatenate([g.ravel() for g in setup.grids])
    out = np.empty(len(points), dtype=np.complex128)
    aw = np.asarray(atoms["w"])
    am = np.asarray(atoms["m"]).astype(np.int64)
    an = np.asarray(atoms["n"]).astype(np.int64)
    ac = np.asarray(atoms["re"]) + 1j * np.asarray(atoms["im"])
    aself = (np.asarray(atoms["flags"]) & 1) == 1
    for i, p in enumerate(np.asarray(points, dtype=np.int64)):
        v = int(np.searchsorted(lay.off, p, side="right") - 1)
        n, m = divmod(int(p - lay.off[v]), lay.MR[v])
        dv = dicts[v]
        acc = complex(res0[p])
        for u in range(W):
            sel = np.nonzero(aw == u)[0]
            if sel.size == 0:
                continue
            K = setup.K[u * W + v]
            du = dicts[u]
            a_c, M_c = K.a_c, K.M_c
            R = M_c // a_c
            s_m = M_c // dv.M
            kp = am[sel] * (M_c // du.M)
            dt = (n * dv.a - an[sel] * du.a) % L
            dt = np.where(dt > L // 2, dt - L, dt)
            nu = dt // a_c
            inb = (nu >= K.nu_lo) & (nu <= K.nu_hi)
            if not inb.any():
                continue
            sel, kp, nu = sel[inb], kp[inb], nu[inb]
            omega = np.exp(2j * np.pi * ((kp * nu) % R) / R)

            def hval(mu):
                mu = mu % M_c
                mu = np.where(2 * mu > M_c, mu - M_c, mu)
                ok = (mu >= K.mu_lo) & (mu <= K.mu_hi)
                vals = np.zeros(mu.shape, dtype=np.complex128)
                vals[ok] = K.h[nu[ok] - K.nu_lo, mu[ok] - K.mu_lo]
                return vals

            zd = ac[sel] * omega * hval(m * s_m - kp)
            zc = ac[sel] * omega * hval(((dv.M - m) % dv.M) * s_m - kp)
            contrib = zd + np.where(aself[sel], 0.0, np.conj(zc))
            acc -= contrib.sum()
        out[i] = acc
    return out


# ---------------------------------------------------------------------------
# O6 initial state bundle
# ---------------------------------------------------------------------------
@dataclass
class Setup:
    dicts: tuple
    thr: float
    Ls: int
    lay: Layout
    grids: list
    K: list
    E0: float
    x: np.ndarray = field(repr=False, default=None)

    @classmethod
    def build(cls, x, dicts, thr, K=None):
        dicts = tuple(dicts)
        lay = layout(dicts, x.size)
        grids = analysis_all(x, dicts, lay)
        if K is None:
            K = kernels(dicts, thr)
        E0 = float(np.dot(x, x))          # E_0 = ||x||^2 (Alg. 1 init)
        return cls(dicts, thr, x.size, lay, grids, K, E0, x)
