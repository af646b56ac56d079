"""Oracle pins: windows, DGT, synthesis (no GPU).

Each test names what pins it: a value the paper or the window formula fixes,
a brute-force definition, or an identity.
"""
import json
import math
import os

import numpy as np
import pytest

from siggen import Dict, HANN, BLACKMAN, GAUSS, random_signal
from oracle import gabor, dense

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_hann_gl4_values():
    # SPEC.md S:56 (derived by direct evaluation of the periodic Hann formula):
    # offsets -2..1 -> {0, .5, 1, .5}, normalised {0, 0.40825, 0.81650, 0.40825}
    j0, g = gabor.window(Dict(HANN, 4, 1, 4))
    assert j0 == -2
    np.testing.assert_allclose(g, [0.0, 0.5 / math.sqrt(1.5), 1.0 / math.sqrt(1.5), 0.5 / math.sqrt(1.5)],
                               atol=1e-15)
    np.testing.assert_allclose(g, [0, 0.40825, 0.81650, 0.40825], atol=1e-5)


@pytest.mark.parametrize("win,gl", [(HANN, 256), (BLACKMAN, 2048), (BLACKMAN, 63), (GAUSS, 101)])
def test_window_unit_norm_peak_at_zero(win, gl):
    # ||g||_2 = 1; zero-phase placement (reading Z1): peak at offset 0
    j0, g = gabor.window(Dict(win, gl, 8, 32))
    assert abs(np.sum(g * g) - 1.0) < 1e-14
    assert int(np.argmax(g)) == -j0


def test_blackman_edge_is_zero():
    # periodic Blackman: 0.42 - 0.5 + 0.08 = 0 at offset -gl/2 (Fig. 1 footprints depend on it)
    j0, g = gabor.window(Dict(BLACKMAN, 64, 16, 64))
    assert abs(g[0]) < 1e-16


TINY = [
    (Dict(HANN, 16, 4, 16),),
    (Dict(HANN, 16, 4, 16), Dict(HANN, 8, 2, 8)),
    (Dict(BLACKMAN, 32, 8, 32), Dict(HANN, 16, 4, 16), Dict(BLACKMAN, 8, 2, 16)),
]


@pytest.mark.parametrize("dicts", TINY)
def test_dgt_equals_bruteforce(dicts):
    # O3 vs the literal definition c = D^H x with materialised atoms (Eq. (3))
    x = random_signal(128, 7)
    lay = gabor.layout(dicts, x.size)
    grids = gabor.analysis_all(x, dicts, lay)
    c = np.concatenate([g.ravel() for g in grids])
    xp = np.zeros(lay.L)
    xp[: x.size] = x
    cb = dense.dgt_bruteforce(xp, dicts)
    assert np.max(np.abs(c - cb)) < 1e-12 * np.linalg.norm(x)


def test_dgt_self_conjugate_bins_real_and_atom_conjugacy():
    # bins 0 and M/2 of a real signal are real; atom(M-m) = conj atom(m)
    d = Dict(BLACKMAN, 32, 8, 32)
    x = random_signal(256, 3)
    c = gabor.dgt(x, d)
    assert np.max(np.abs(c[:, 0].imag)) < 1e-13
    assert np.max(np.abs(c[:, 16].imag)) < 1e-13
    for m in (1, 5, 13):
        np.testing.assert_allclose(dense.atom(d, 32 - m, 3, 256), np.conj(dense.atom(d, m, 3, 256)),
                                   atol=1e-15)


def test_dgt_gl_longer_than_M_folds():
    # gl > M (Gaussian support) folds j mod M; still equals D^H x
    d = Dict(GAUSS, 41, 4, 16)
    x = random_signal(128, 11)
    c = gabor.dgt(x, d).ravel()
    cb = dense.dgt_bruteforce(x, (d,))
    assert np.max(np.abs(c - cb)) < 1e-12


def test_layout_padding_c2():
    # reading Z3: Ls=220500 padded to a multiple of lcm{a_w, M_w} = 4096 -> 221184
    from siggen import CONFIGS
    lay = gabor.layout(CONFIGS["C2"].dicts, 220500)
    assert lay.L == 221184
    assert lay.N == [3456, 1728, 864, 432, 216]
    assert lay.MR == [129, 257, 513, 1025, 2049]
    assert lay.P == 2_218_536


def test_layout_rejects_incompatible():
    # P:296-303 compatibility; SPEC S:63 example (96 does not divide 128)
    with pytest.raises(ValueError):
        gabor.layout((Dict(HANN, 384, 96, 384), Dict(HANN, 512, 128, 512)), 4096)
    with pytest.raises(ValueError):
        gabor.layout((Dict(HANN, 100, 30, 100),), 3000)      # M/a not integer


def _atoms(rows):
    from oracle.loop import ATOM_DTYPE
    return np.array(rows, dtype=ATOM_DTYPE)


def test_synthesis_single_coefficient_is_window():
    # Eq. (18): a single self-conjugate coefficient c(0,0)=1 synthesises the window itself
    d = Dict(HANN, 16, 4, 16)
    y = gabor.synthesize(_atoms([(0, 0, 0, 1, 1.0, 0.0)]), (d,), 64)
    j0, g = gabor.window(d)
    ref = np.zeros(64)
    ref[(np.arange(g.size) + j0) % 64] = g
    np.testing.assert_allclose(y, ref, atol=1e-16)


@pytest.mark.parametrize("dicts", TINY[1:])
def test_synthesis_adjoint_identity(dicts):
    # <synth(c), y> = sum over atoms of (1 or 2) * Re(c * conj(<y, d>)) (Eq. (18))
    rng = np.random.Generator(np.random.PCG64(5))
    L = 128
    lay = gabor.layout(dicts, L)
    rows = []
    for _ in range(40):
        w = int(rng.integers(0, len(dicts)))
        m = int(rng.integers(0, lay.MR[w]))
        n = int(rng.integers(0, lay.N[w]))
        sc = int(m == 0 or 2 * m == dicts[w].M)
        rows.append((w, m, n, sc, rng.normal(), 0.0 if sc else rng.normal()))
    at = _atoms(rows)
    y = random_signal(L, 9)
    s = gabor.synthesize(at, dicts, L)
    cy = dense.dgt_bruteforce(y, dicts)
    rhs = 0.0
    for a in at:
        p = lay.off[a["w"]] + a["n"] * lay.MR[a["w"]] + a["m"]
        mult = 1.0 if a["flags"] else 2.0
        rhs += mult * np.real((a["re"] + 1j * a["im"]) * np.conj(cy[p]))
    assert abs(np.dot(s, y) - rhs) < 1e-12 * max(1.0, abs(rhs))
