"""Oracle pins for the coefficient-domain MP loop (no GPU).

* eps = 0: the kernel loop reproduces exact signal-domain MP (Eq. (8))
  and the literal dense Alg. 1 with the full Gram (SPEC acceptance 3).
* eps > 0: the kernel loop (fold rule Z14) equals literal dense Alg. 1 run with the
  explicitly thresholded G_eps over the full complex dictionary (Eq. (9)).
* Eq. (19)/(20) against a 2x2 least-squares projection on materialised atoms.
* signal MP conserves energy (Eq. (5)).
* the frame/group max cache equals a full scan (O11).
"""
import math

import numpy as np
import pytest

from siggen import Dict, HANN, BLACKMAN, CONFIGS, random_signal, signal
import oracle
from oracle import dense, gabor, loop


def _seq(a):
    return list(zip(a["w"].tolist(), a["m"].tolist(), a["n"].tolist()))


CASES = [
    ((Dict(BLACKMAN, 64, 16, 64),), 512, 100),                         # SPEC acceptance 3
    ((Dict(HANN, 16, 4, 16), Dict(HANN, 8, 2, 8)), 96, 60),
    ((Dict(BLACKMAN, 32, 8, 32), Dict(HANN, 16, 4, 16), Dict(BLACKMAN, 8, 2, 16)), 128, 80),
]


@pytest.mark.parametrize("dicts,L,steps", CASES)
def test_threshold_zero_equals_signal_mp_and_dense(dicts, L, steps):
    x = random_signal(L, 21)
    S = oracle.Setup.build(x, dicts, 0.0)
    r = loop.mp_run(S, steps)
    a_s, e_s, te_s, _, _ = dense.signal_mp(x, dicts, steps)
    a_d, e_d, _, _ = dense.dense_alg1(x, dicts, 0.0, steps)
    assert _seq(r.atoms) == _seq(a_s) == _seq(a_d)
    np.testing.assert_allclose(r.atoms["re"], a_s["re"], atol=1e-12)
    np.testing.assert_allclose(r.atoms["im"], a_s["im"], atol=1e-12)
    assert np.max(np.abs(r.energy - e_s)) < 1e-12 * S.E0
    assert np.max(np.abs(r.energy - te_s)) < 1e-12 * S.E0      # estimate == true energy at eps=0


@pytest.mark.parametrize("thr", [1e-4, 1e-2, 1e-1])
@pytest.mark.parametrize("dicts,L,steps", CASES[1:] + [
    ((Dict(BLACKMAN, 64, 8, 64), Dict(BLACKMAN, 128, 32, 128), Dict(BLACKMAN, 32, 8, 32)), 512, 200)])
def test_truncated_equals_dense_alg1(thr, dicts, L, steps):
    x = random_signal(L, 5)
    S = oracle.Setup.build(x, dicts, thr)
    r = loop.mp_run(S, steps)
    a_d, e_d, _, cres = dense.dense_alg1(x, dicts, thr, steps)
    assert _seq(r.atoms) == _seq(a_d)
    assert np.max(np.abs(r.energy - e_d)) < 1e-12 * S.E0
    assert np.max(np.abs(r.res - cres)) < 1e-11 * math.sqrt(S.E0)


def test_pair_adjustment_is_least_squares():
    # Eq. (19) / (20): c~ and conj(c~) solve min ||r - a d - b conj(d)||, and E~ is the
    # energy that projection removes (brute force on materialised atoms; App. A3)
    d = Dict(HANN, 8, 2, 32)
    L = 64
    checked = 0
    for k in range(1, 16):
        at = dense.atom(d, k, 5, L)
        if abs(np.sum(at * at)) < 1e-3:  # rho = <d, conj d> must be non-negligible
            continue
        x = 2.0 * np.real((0.1 + 0.8j) * at) + 1e-3 * random_signal(L, k)
        S = oracle.Setup.build(x, (d,), 0.0)
        r = loop.mp_run(S, 1)
        a = r.atoms[0]
        if (a["m"], a["n"], a["flags"]) != (k, 5, 0):
            continue
        checked += 1
        dd = dense.atom(d, int(a["m"]), int(a["n"]), L)
        B = np.stack([dd, np.conj(dd)], axis=1)
        coef, *_ = np.linalg.lstsq(B, x.astype(np.complex128), rcond=None)
        ct = a["re"] + 1j * a["im"]
        assert abs(coef[0] - ct) < 1e-12 and abs(coef[1] - np.conj(ct)) < 1e-12
        resid = x - B @ coef
        Et = S.E0 - r.energy[1]
        assert abs((np.dot(x, x) - np.vdot(resid, resid).real) - Et) < 1e-12 * S.E0
    assert checked >= 2


def test_signal_mp_conserves_energy():
    # ||x||^2 = ||r_K||^2 + sum E~ and ||r_k|| decreasing (exact MP, Eq. (5))
    dicts = CASES[2][0]
    x = random_signal(128, 2)
    at, e, te, stop, rK = dense.signal_mp(x, dicts, 120)
    Et = -np.diff(e)
    assert abs(np.dot(x, x) - (np.dot(rK, rK) + Et.sum())) < 1e-12 * np.dot(x, x)
    assert np.all(np.diff(te) <= 1e-15 * te[0])


def test_maxcache_equals_full_scan():
    # O11: frame/group max cache == plain scan over every coefficient, identical runs
    for cfg, steps in ((CONFIGS["C0"], 500), (CONFIGS["C1"], 1500)):
        x = signal(cfg)
        S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
        r1 = loop.mp_run(S, steps)
        r2 = loop.mp_run(S, steps, full_scan=True)
        assert np.array_equal(r1.index, r2.index)
        assert np.array_equal(r1.energy, r2.energy)


def _bruteforce_gap(res):
    # (s1 - s2)/s1 of the plain score |c^|^2 over every coefficient, s2 over p != argmax
    s = res.real * res.real + res.imag * res.imag
    p = int(np.argmax(s))
    s1 = s[p]
    s[p] = -1.0
    return (s1 - s.max()) / s1


@pytest.mark.parametrize("full_scan", [False, True])
def test_gaps_equal_bruteforce_second_best(full_scan):
    # the near-tie gap gap_k = (s1 - s2)/s1 that decides the fp32
    # acceptance: at sampled k it equals a brute-force second-best over the residual that
    # the loop holds before selection k (a run stopped after k selections), in both the
    # max-cache and the full-scan mode
    for cfg, ks in ((CONFIGS["C0"], (0, 1, 7, 60, 233, 499)), (CONFIGS["C1"], (0, 5, 111, 640))):
        x = signal(cfg)
        S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
        steps = ks[-1] + 1
        r = loop.mp_run(S, steps, full_scan=full_scan)
        assert r.n == steps
        for k in ks:
            rk = loop.mp_run(S, k, want_gaps=False)
            assert r.gaps[k] == _bruteforce_gap(rk.res)


def test_gaps_see_an_exact_tie():
    # two identical separated atoms: the first selection has a gap of exactly 0
    d = Dict(HANN, 16, 4, 16)
    L = 128
    x = 2 * np.real(dense.atom(d, 3, 4, L)) + 2 * np.real(dense.atom(d, 3, 20, L))
    S = oracle.Setup.build(x, (d,), 1e-4)
    for fs in (False, True):
        assert loop.mp_run(S, 2, full_scan=fs).gaps[0] == 0.0


def test_tie_break_lowest_index():
    # Z10: exact ties go to the lowest global index.  Two identical well separated
    # pair atoms in the same dictionary -> the earlier frame is selected first.
    d = Dict(HANN, 16, 4, 16)
    L = 128
    x = 2 * np.real(dense.atom(d, 3, 4, L)) + 2 * np.real(dense.atom(d, 3, 20, L))
    S = oracle.Setup.build(x, (d,), 1e-4)
    s = np.abs(S.grids[0]) ** 2
    assert s[4, 3] == s[20, 3]            # the tie is exact in the DGT
    r = loop.mp_run(S, 2)
    assert (r.atoms["n"][0], r.atoms["m"][0]) == (4, 3)


def test_stop_rules():
    d = (Dict(HANN, 16, 4, 16),)
    z = np.zeros(64)
    S = oracle.Setup.build(z, d, 1e-4)
    assert loop.mp_run(S, 10).stop_name == "zero"                # max score 0
    assert loop.mp_run(S, 10, errdb=-40).stop_name == "errtol"   # E_0 = 0 <= tol
    x = random_signal(64, 1)
    S = oracle.Setup.build(x, d, 1e-4)
    r = loop.mp_run(S, 10**6, errdb=-20)
    assert r.stop_name == "errtol"
    assert r.energy[-1] <= 1e-2 * S.E0 < r.energy[-2]
    assert loop.mp_run(S, 0).n == 0
    # large threshold: the estimate eventually goes negative -> E_k < 0 stop
    S = oracle.Setup.build(random_signal(256, 4), (Dict(HANN, 16, 4, 16), Dict(HANN, 32, 8, 32)), 0.3)
    r = loop.mp_run(S, 10**5)
    assert r.stop_name == "negest" and r.energy[-1] < 0 <= r.energy[-2]


def test_c0_recovers_planted_atoms_and_estimate_tracks_truth():
    # config-scale self-consistency (parity unpinned at this scale):
    # the E_k estimate follows the true residual energy and the 20 planted
    # atoms dominate the first selections.
    cfg = CONFIGS["C0"]
    x = signal(cfg)
    S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
    r = loop.mp_run(S, cfg.maxit)
    assert r.stop_name == "maxit" and r.n == 500
    y = gabor.synthesize(r.atoms, cfg.dicts, S.lay.L, cfg.Ls)
    true_db = 10 * np.log10(np.sum((x - y) ** 2) / S.E0)
    est_db = 10 * np.log10(r.energy[-1] / S.E0)
    assert abs(true_db - est_db) < 1.0
    assert np.all(np.diff(r.energy) <= 0)


def test_residual_at_one_by_one_equals_loop():
    # the single-coefficient restatement of Alg. 3 (gabor.residual_at) reproduces the
    # loop's residual; it is what the GPU tests use for sampled full-size checks
    cfg = CONFIGS["C1"]
    x = signal(cfg)
    S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
    r = loop.mp_run(S, 2000)
    rng = np.random.default_rng(3)
    pts = np.unique(np.clip(np.concatenate([r.index[-40:], r.index[-40:] + 1, r.index[-40:] - 2,
                                            rng.integers(0, S.lay.P, 40)]), 0, S.lay.P - 1))
    got = gabor.residual_at(S, r.atoms, pts)
    assert np.max(np.abs(got - r.res[pts])) < 1e-14 * math.sqrt(S.E0)


# ---------------------------------------------------------------------------
# Alg. 2: approximate coefficient-domain MP nested in resets
# ---------------------------------------------------------------------------
def _dense_energy(x, dicts, atoms, L):
    """||x_pad - sum_atoms||^2 with materialised atoms (independent of gabor.synthesize):
    c~ d for self-conjugate atoms, 2 Re(c~ d) for pairs (Eq. (18))."""
    r = np.zeros(L)
    r[: x.size] = x
    for a in atoms:
        d = dense.atom(dicts[int(a["w"])], int(a["m"]), int(a["n"]), L)
        z = (a["re"] + 1j * a["im"]) * d
        r -= z.real if a["flags"] & 1 else 2.0 * z.real
    return float(np.dot(r, r))


def test_reset_without_reset_equals_alg1():
    cfg = CONFIGS["C0"]
    x = signal(cfg)
    r1 = loop.mp_run(oracle.Setup.build(x, cfg.dicts, cfg.thr), 300, cfg.errdb)
    r2 = loop.mp_run_reset(x, cfg.dicts, cfg.thr, 300, cfg.errdb, reset_every=10**6)
    assert r2.passes == 1 and r2.n == r1.n
    assert r1.atoms.tobytes() == r2.atoms.tobytes() and np.array_equal(r1.energy, r2.energy)


@pytest.mark.parametrize("every", [1, 7, 25])
def test_reset_threshold_zero_equals_signal_mp(every):
    # eps = 0: every pass is exact MP, so resets change nothing but rounding (Eq. (8))
    dicts = (Dict(HANN, 16, 4, 16), Dict(HANN, 8, 2, 8))
    x = random_signal(96, 21)
    r = loop.mp_run_reset(x, dicts, 0.0, 60, -math.inf, every)
    a_s, e_s, _, _, _ = dense.signal_mp(x, dicts, 60)
    assert _seq(r.atoms) == _seq(a_s)
    np.testing.assert_allclose(r.atoms["re"], a_s["re"], atol=1e-12)
    np.testing.assert_allclose(r.energy, e_s, rtol=0, atol=1e-12 * e_s[0])


def test_reset_pass_energies_are_true_residual_energies():
    # at every pass start E_k = ||x - D c_out||^2 (Alg. 2 step 2d), recomputed from the
    # atom list with materialised atoms; inside a pass E_k is the Eq. (20) estimate
    dicts = (Dict(BLACKMAN, 32, 8, 32), Dict(HANN, 16, 4, 16))
    x = random_signal(200, 5)          # ragged: padded to L = 224 (reading Z3)
    lay = gabor.layout(dicts, x.size)
    every = 9
    r = loop.mp_run_reset(x, dicts, 1e-2, 45, -math.inf, every)
    assert r.n == 45 and r.passes == 5
    for k in range(0, r.n, every):
        assert abs(r.energy[k] - _dense_energy(x, dicts, r.atoms[:k], lay.L)) <= 1e-11 * r.energy[0]
    assert abs(float(np.dot(r.residual, r.residual)) - _dense_energy(x, dicts, r.atoms, lay.L)) <= 1e-11 * r.energy[0]


def test_reset_recovers_truncation_drift():
    # Theorem 2: with a coarse Gram threshold the plain approximate loop
    # stalls above the exact error, the reset loop keeps decreasing the true error
    dicts = (Dict(HANN, 32, 8, 32), Dict(HANN, 16, 4, 16))
    x = random_signal(256, 3)
    lay = gabor.layout(dicts, x.size)
    K = 150
    plain = loop.mp_run(oracle.Setup.build(x, dicts, 0.3), K)
    reset = loop.mp_run_reset(x, dicts, 0.3, K, -math.inf, 10)
    e_plain = _dense_energy(x, dicts, plain.atoms, lay.L)
    e_reset = float(np.dot(reset.residual, reset.residual))
    assert e_reset < 0.5 * e_plain
    # the true energies at the pass starts decrease
    starts = reset.energy[::10][: reset.passes]
    assert np.all(np.diff(starts) < 0)


# ---------------------------------------------------------------------------
# pedantic selection: argmax of the energy the selection removes
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("dicts,L,steps", CASES[1:])
def test_pedantic_threshold_zero_equals_bruteforce_projection_mp(dicts, L, steps):
    # eps = 0: the pedantic coefficient-domain loop (Eq. (19)/(20) scores) equals MP that
    # selects by the least-squares projection energy onto span{d, conj d} of materialised atoms
    x = random_signal(L, 23)
    S = oracle.Setup.build(x, dicts, 0.0)
    r = loop.mp_run(S, steps, pedantic=True)
    idx, e = dense.signal_mp_pedantic(x, dicts, steps)
    assert np.array_equal(r.index, idx)
    np.testing.assert_allclose(r.energy, e, rtol=0, atol=1e-11 * e[0])


def test_pedantic_maxcache_equals_full_scan_and_differs_from_plain():
    cfg = CONFIGS["C0"]
    x = signal(cfg)
    S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
    a = loop.mp_run(S, 300, cfg.errdb, pedantic=True)
    b = loop.mp_run(S, 300, cfg.errdb, pedantic=True, full_scan=True)
    c = loop.mp_run(S, 300, cfg.errdb)
    assert np.array_equal(a.index, b.index) and np.array_equal(a.energy, b.energy)
    assert not np.array_equal(a.index, c.index)          # the rule matters on C0 (low bins)
    assert a.energy[-1] <= c.energy[-1]                   # and removes at least as much energy here
