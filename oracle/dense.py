"""Tiny-scale dense oracle layer (TEST INFRASTRUCTURE ONLY), numpy fp64.

Materialised atoms (Eq. (3)), brute-force analysis D^H x, dense Gram matrices
G = D^H D, exact signal-domain MP (P:317-341 with the real-atom
rules Eqs. (18)-(20)), and the literal dense Alg. 1 run with the
hard-thresholded Gram G_eps (Eq. (7)) over the full complex
dictionary with real-atom pairs -- SURVEY.md §8(c) O9/O10.  Size-guarded.
"""
from __future__ import annotations

import math

import numpy as np

from .gabor import window, layout
from .loop import ATOM_DTYPE, error_tolerance

MAX_L = 2048


def _guard(L):
    if L > MAX_L:
        raise ValueError(f"dense oracle refuses L={L} > {MAX_L}")


def atom(d, m, n, L):
    """d_{m+nM}(l) = g(l - na) e^{i 2 pi m (l - na)/M}, l - na taken as the signed
    window offset, positions circular mod L (Eq. (3))."""
    j0, g = window(d)
    j = j0 + np.arange(g.size)
    v = np.zeros(L, dtype=np.complex128)
    np.add.at(v, (n * d.a + j) % L, g * np.exp(2j * np.pi * m * j / d.M))
    return v


def dictionary(dicts, L, full=False):
    """Columns ordered (w, n, m); m over 0..floor(M/2) (reduced) or 0..M-1."""
    _guard(L)
    cols = []
    for d in dicts:
        nb = d.M if full else d.M // 2 + 1
        for n in range(L // d.a):
            for m in range(nb):
                cols.append(atom(d, m, n, L))
    return np.stack(cols, axis=1)


def dgt_bruteforce(x, dicts):
    """c = D^H x on the reduced dictionary (Alg. 1 init)."""
    return dictionary(dicts, x.size).conj().T @ x


def gram(dicts, L):
    """G(q, p) = <d_p, d_q> = (D^H D)(q, p), full complex dictionary."""
    D = dictionary(dicts, L, full=True)
    return D.conj().T @ D


def _pair_step(c, rho):
    """Eq. (19) with reading Z11 (conj(rho)) and Eq. (20)."""
    ct = (c - np.conj(rho) * np.conj(c)) / (1.0 - abs(rho) ** 2)
    X, Y = ct.real, ct.imag
    Et = 2.0 * (X * X + Y * Y + rho.real * (X * X - Y * Y) - 2.0 * rho.imag * X * Y)
    return ct, Et


def signal_mp(x, dicts, maxit, errdb=-math.inf):
    """Exact MP in the signal domain: c = D^H r recomputed every step,
    same selection / tie / real-atom rules as the coefficient-domain loop."""
    dicts = tuple(dicts)
    lay = layout(dicts, x.size)
    L = lay.L
    _guard(L)
    r = np.zeros(L)
    r[: x.size] = x
    D = dictionary(dicts, L)
    E0 = float(np.dot(x, x))
    tol = error_tolerance(errdb, E0)
    E = E0
    atoms, energy, true_energy = [], [E0], [E0]
    stop = 0
    while True:
        if len(atoms) >= maxit:
            stop = 1; break
        if E <= tol:
            stop = 2; break
        if E < 0:
            stop = 3; break
        c = D.conj().T @ r
        s = c.real * c.real + c.imag * c.imag
        p = int(np.argmax(s))                      # first maximum = lowest index
        if not s[p] > 0:
            stop = 4; break
        w = int(np.searchsorted(lay.off, p, side="right") - 1)
        n, k = divmod(p - lay.off[w], lay.MR[w])
        d = D[:, p]
        if k == 0 or 2 * k == dicts[w].M:
            ct = complex(c[p].real, 0.0)
            Et = ct.real * ct.real
            r = r - ct.real * d.real
            flags = 1
        else:
            rho = complex(np.sum(d * d))              # <d, conj d>
            ct, Et = _pair_step(c[p], rho)
            r = r - 2.0 * np.real(ct * d)
            flags = 0
        E = E - Et
        atoms.append((w, k, n, flags, ct.real, ct.imag))
        energy.append(E)
        true_energy.append(float(np.dot(r, r)))
    return (np.array(atoms, dtype=ATOM_DTYPE), np.array(energy), np.array(true_energy), stop, r)


def threshold_gram(G, dicts, L, thr):
    """G_eps per (cross-)Gram block, relative to each block's own max (Eq. (7), Z5/Z6)."""
    Ge = np.zeros_like(G)
    offs = [0]
    for d in dicts:
        offs.append(offs[-1] + d.M * (L // d.a))
    for a in range(len(dicts)):
        for b in range(len(dicts)):
            blk = G[offs[a]:offs[a + 1], offs[b]:offs[b + 1]]
            mx = np.abs(blk).max()
            Ge[offs[a]:offs[a + 1], offs[b]:offs[b + 1]] = np.where(np.abs(blk) > thr * mx, blk, 0)
    return Ge, offs


def dense_alg1(x, dicts, thr, maxit, errdb=-math.inf):
    """Literal Alg. 1 with G_eps (Eq. (9) recursion P:424-434) over the
    full complex dictionary; real atoms are the pair {d, conj d}:
        c^ <- c^ - c~ G_eps(., p) - conj(c~) G_eps(., p_conj)   (pair)
        c^ <- c^ - c~ G_eps(., p)                               (self-conjugate)
    with rho = G_eps(p_conj, p); selection over the reduced positions."""
    dicts = tuple(dicts)
    lay = layout(dicts, x.size)
    L = lay.L
    _guard(L)
    xp = np.zeros(L)
    xp[: x.size] = x
    G = gram(dicts, L)
    Ge, foff = threshold_gram(G, dicts, L, thr)
    Dfull = dictionary(dicts, L, full=True)
    c = Dfull.conj().T @ xp
    # reduced position -> full index
    red = []
    for w, d in enumerate(dicts):
        for n in range(L // d.a):
            for m in range(d.M // 2 + 1):
                red.append(foff[w] + n * d.M + m)
    red = np.array(red)
    E0 = float(np.dot(x, x))
    tol = error_tolerance(errdb, E0)
    E = E0
    atoms, energy = [], [E0]
    stop = 0
    while True:
        if len(atoms) >= maxit:
            stop = 1; break
        if E <= tol:
            stop = 2; break
        if E < 0:
            stop = 3; break
        cr = c[red]
        s = cr.real * cr.real + cr.imag * cr.imag
        p = int(np.argmax(s))
        if not s[p] > 0:
            stop = 4; break
        w = int(np.searchsorted(lay.off, p, side="right") - 1)
        n, k = divmod(p - lay.off[w], lay.MR[w])
        M = dicts[w].M
        pf = foff[w] + n * M + k
        if k == 0 or 2 * k == M:
            ct = complex(cr[p].real, 0.0)
            Et = ct.real * ct.real
            c = c - ct * Ge[:, pf]
            flags = 1
        else:
            pc = foff[w] + n * M + (M - k) % M
            rho = complex(Ge[pc, pf])
            ct, Et = _pair_step(cr[p], rho)
            c = c - ct * Ge[:, pf] - np.conj(ct) * Ge[:, pc]
            flags = 0
        E = E - Et
        atoms.append((w, k, n, flags, ct.real, ct.imag))
        energy.append(E)
    return np.array(atoms, dtype=ATOM_DTYPE), np.array(energy), stop, c[red]


def signal_mp_pedantic(x, dicts, maxit):
    """Exact signal-domain MP with the pedantic selection rule, by brute
    force: every step projects the residual onto span_R{Re d_p, Im d_p} (the real
    atom pair d_p, conj d_p) for every reduced p by least squares on the materialised
    atoms, selects the largest projection energy (ties -> lowest p) and subtracts the
    projection.  Independent of Eqs. (19)/(20).  Returns (index[steps], energy[steps+1])."""
    dicts = tuple(dicts)
    lay = layout(dicts, x.size)
    L = lay.L
    _guard(L)
    r = np.zeros(L)
    r[: x.size] = x
    D = dictionary(dicts, L)
    bases = []
    for p in range(D.shape[1]):
        d = D[:, p]
        B = np.stack([d.real, d.imag], axis=1) if np.linalg.norm(d.imag) > 1e-12 * np.linalg.norm(d.real) else d.real[:, None]
        Q, _ = np.linalg.qr(B)
        bases.append(Q)
    idx, energy = [], [float(np.dot(r, r))]
    for _ in range(maxit):
        en = np.array([float(np.sum((Q.T @ r) ** 2)) for Q in bases])
        p = int(np.argmax(en))
        if not en[p] > 0:
            break
        Q = bases[p]
        r = r - Q @ (Q.T @ r)
        idx.append(p)
        energy.append(float(np.dot(r, r)))
    return np.asarray(idx, dtype=np.int64), np.asarray(energy)
