"""Oracle pins for the Gram (cross-)kernels (no GPU)."""
import json
import math
import os

import numpy as np
import pytest

from siggen import Dict, HANN, BLACKMAN, GAUSS, CONFIGS
from oracle import gabor, dense

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _gauss_gl(a, M, rel=1e-10):
    # Gaussian support: every offset where exp(-pi j^2/(aM)) exceeds 1e-10 (reading Z2, O2)
    jmax = int(math.floor(math.sqrt(-math.log(rel) * a * M / math.pi)))
    return 2 * jmax + 2          # offsets -(jmax+1) .. jmax


def test_fig1_footprints_paper_values():
    # PAPER Fig. 1: Gaussian 9x9, Hann 31x7, Blackman 23x7 at a=512, M=2048, -80 dB
    gold = json.load(open(os.path.join(GOLDEN, "fig1_footprints.json")))
    a, M, thr = gold["a"], gold["M"], gold["relative_threshold"]
    kinds = {"hann": (HANN, M), "blackman": (BLACKMAN, M), "gauss": (GAUSS, _gauss_gl(a, M))}
    for name, (win, gl) in kinds.items():
        d = Dict(win, gl, a, M)
        K = gabor.cross_kernel(d, d, thr)
        got = [K.mu_hi - K.mu_lo + 1, K.nu_hi - K.nu_lo + 1]
        assert got == gold["footprints_freq_by_time"][name], name


def test_gauss_closed_form():
    # App. A5 of SURVEY.md: for g ~ exp(-pi t^2/(aM)),
    # h(mu, nu) = exp(-(pi a / 2M)(mu^2 + nu^2)) e^{i pi a mu nu / M}; |h| > 1e-4 <=> mu^2+nu^2 < 23.45
    a, M = 512, 2048
    d = Dict(GAUSS, _gauss_gl(a, M), a, M)
    K = gabor.cross_kernel(d, d, 1e-4)
    for mu in range(K.mu_lo, K.mu_hi + 1):
        for nu in range(K.nu_lo, K.nu_hi + 1):
            ref = math.exp(-(math.pi * a / (2 * M)) * (mu * mu + nu * nu)) * \
                np.exp(1j * math.pi * a * mu * nu / M)
            got = K.h[nu - K.nu_lo, mu - K.mu_lo]
            if mu * mu + nu * nu < 23.45:
                assert abs(got - ref) < 1e-10, (mu, nu)
            else:
                assert got == 0
    assert K.kept == sum(1 for mu in range(-5, 6) for nu in range(-5, 6) if mu * mu + nu * nu < 23.45) == 69


def _dense_cross_check(du, dv, L):
    """Every entry <d^u_{k,j}, d^v_{m,n}> of the dense cross-Gram equals the kernel formula
    h_{u,v}(m' - k', nu) omega_R^{k' nu}  (Eq. (14) P:554 single, Eq. (17) P:631 cross;
    App. A1-A2), untruncated kernel."""
    K = gabor.cross_kernel(du, dv, 0.0)
    Du = dense.dictionary((du,), L, full=True)
    Dv = dense.dictionary((dv,), L, full=True)
    G = Dv.conj().T @ Du                       # G[(m,n), (k,j)] = <d_{k,j}, d_{m,n}>
    a_c, M_c = K.a_c, K.M_c
    R = M_c // a_c
    Nu, Nv = L // du.a, L // dv.a
    err = 0.0
    for j in range(Nu):
        for k in range(du.M):
            kp = k * (M_c // du.M)
            col = G[:, j * du.M + k]
            for n in range(Nv):
                dt = n * dv.a - j * du.a
                # circular time lag on the common grid, signed nearest representative
                dt = (dt + L // 2) % L - L // 2
                nu = dt // a_c
                for m in range(dv.M):
                    mp = m * (M_c // dv.M)
                    pred = gabor.kernel_value(K, mp - kp, nu) * np.exp(2j * np.pi * ((kp * nu) % R) / R)
                    err = max(err, abs(col[n * dv.M + m] - pred))
    return err


@pytest.mark.parametrize("du,dv,L", [
    (Dict(HANN, 16, 4, 16), Dict(HANN, 16, 4, 16), 64),
    (Dict(HANN, 16, 4, 16), Dict(HANN, 8, 2, 8), 64),
    (Dict(HANN, 8, 2, 8), Dict(HANN, 16, 4, 16), 64),
    (Dict(BLACKMAN, 32, 4, 32), Dict(BLACKMAN, 16, 2, 8), 96),
    (Dict(BLACKMAN, 16, 2, 8), Dict(BLACKMAN, 32, 8, 32), 96),
])
def test_cross_gram_reconstruction(du, dv, L):
    assert _dense_cross_check(du, dv, L) < 1e-13


def test_spec_acceptance_gram_blackman_32_128():
    # SPEC acceptance 1 sizes: L=1024, Blackman a=32, M=128, 50 random columns
    d = Dict(BLACKMAN, 128, 32, 128)
    L = 1024
    K = gabor.cross_kernel(d, d, 0.0)
    D = dense.dictionary((d,), L, full=True)
    rng = np.random.Generator(np.random.PCG64(1))
    R = K.M_c // K.a_c
    for _ in range(50):
        k, j = int(rng.integers(0, 128)), int(rng.integers(0, L // 32))
        col = D.conj().T @ D[:, j * 128 + k]
        for n in range(L // 32):
            nu = ((n - j) + (L // 32) // 2) % (L // 32) - (L // 32) // 2
            ph = np.exp(2j * np.pi * ((k * nu) % R) / R)
            pred = np.array([gabor.kernel_value(K, m - k, nu) for m in range(128)]) * ph
            assert np.max(np.abs(col[n * 128:(n + 1) * 128] - pred)) < 1e-12


def test_auto_kernel_invariants_and_symmetry():
    # h_uu(0,0) = 1 (unit-norm window), max|h_uu| = 1; conjugate symmetric about both
    # axes: h(-mu,nu) = h(mu,-nu) = conj h(mu,nu)
    for d in (Dict(HANN, 256, 64, 256), Dict(BLACKMAN, 2048, 256, 4096)):
        K = gabor.cross_kernel(d, d, 0.0)
        assert abs(gabor.kernel_value(K, 0, 0) - 1.0) < 1e-14
        assert abs(K.mx - 1.0) < 1e-14
        for mu, nu in [(1, 0), (3, 1), (7, 2), (2, -3)]:
            h = gabor.kernel_value(K, mu, nu)
            assert abs(gabor.kernel_value(K, -mu, nu) - np.conj(h)) < 1e-15
            assert abs(gabor.kernel_value(K, mu, -nu) - np.conj(h)) < 1e-15


def test_threshold_is_strict_relative_and_monotone():
    # Eq. (7) strict '>' relative to the kernel's own max (Z5, Z6); raising eps never grows the box
    du, dv = Dict(BLACKMAN, 256, 64, 256), Dict(BLACKMAN, 1024, 256, 1024)
    prev = None
    for thr in (1e-6, 1e-5, 1e-4, 1e-3, 1e-2):
        K = gabor.cross_kernel(du, dv, thr)
        mag = np.abs(K.h)
        assert np.all((mag == 0) | (mag > thr * K.mx))
        box = (K.mu_hi - K.mu_lo + 1) * (K.nu_hi - K.nu_lo + 1)
        if prev is not None:
            assert box <= prev
        prev = box
    # all four box edges hold a kept entry (minimal box)
    assert np.any(K.h[0] != 0) and np.any(K.h[-1] != 0)
    assert np.any(K.h[:, 0] != 0) and np.any(K.h[:, -1] != 0)


def test_kernel_storage_configs():
    # regression of SURVEY.md App. B (computed there independently): stored box entries
    want = {"C0": 217, "C1": 4641, "C2": 78117}
    for c, n in want.items():
        K = gabor.kernels(CONFIGS[c].dicts, CONFIGS[c].thr)
        assert sum(k.h.size for k in K) == n
