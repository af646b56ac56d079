"""Seeded synthetic inputs and workload configs (generator ``v1``).

This module is shared by the oracle tests and the CUDA-path tests/bench, so it
deliberately contains *none* of the matching-pursuit arithmetic: no DGT, no
Gram kernels, no selection or update.  It only builds signals and lists the
dictionary/stop parameters of BASELINE.json ``configs[0..4]`` (C0..C4).

The paper measures on SQAM track 39, a 137 s piano recording at 44.1 kHz
(PAPER.md P:1038-1039), which is not available here.  The audio-like generator
``audio_like`` stands in for it (SURVEY.md §8(d) recipe; DESIGN.md §3 lists
every choice made where BASELINE.json is silent).

All randomness comes from ``numpy.random.Generator(PCG64(seed))``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GENERATOR_VERSION = "v1"
FS = 44100

HANN, BLACKMAN, GAUSS = 1, 2, 3
WINDOW_NAMES = {HANN: "hann", BLACKMAN: "blackman", GAUSS: "gauss"}


@dataclass(frozen=True)
class Dict:
    """One Gabor dictionary (window kind, window length gl, hop a, channels M).

    Mirrors ``dgtrealmp_parbuf_add_firwin(win, gl, a, M)``.
    """

    win: int
    gl: int
    a: int
    M: int


@dataclass(frozen=True)
class Config:
    name: str
    Ls: int
    dicts: tuple
    thr: float
    maxit: int
    errdb: float
    seed: int
    signal: str  # which generator builds x
    precisions: tuple = ("f64",)
    note: str = ""


def _blackman_set(widths, hop_div, m_mul):
    return tuple(Dict(BLACKMAN, w, w // hop_div, w * m_mul) for w in widths)


# BASELINE.json configs[0..4]; stop rules per SURVEY.md §8(d) table.
CONFIGS = {
    "C0": Config("C0", 4096, (Dict(HANN, 256, 64, 256),), 1e-4, 500, -math.inf, 0,
                 "planted_c0", ("f64", "f32")),
    "C1": Config("C1", 65536, _blackman_set((512, 1024, 2048), 4, 1), 1e-4, 10_000,
                 -math.inf, 1, "planted_c1", ("f64", "f32")),
    "C2": Config("C2", 220500, _blackman_set((256, 512, 1024, 2048, 4096), 4, 1), 1e-4,
                 100_000, -40.0, 2, "audio_like", ("f64", "f32"),
                 "run until 40 dB SNR (E_k <= 1e-4 E_0) or 1e5 atoms"),
    "C3": Config("C3", 220500, _blackman_set((256, 512, 1024, 2048, 4096), 8, 2), 1e-5,
                 200_000, -math.inf, 2, "audio_like", ("f64", "f32")),
    "C4": Config("C4", 1 << 22,
                 _blackman_set((128, 256, 512, 1024, 2048, 4096, 8192, 16384), 4, 1), 1e-6,
                 1_000_000, -math.inf, 1000, "audio_tiled", ("f64", "f32")),
}


# ----------------------------------------------------------------------------
# planted-atom signals (C0, C1)
# ----------------------------------------------------------------------------
def _planted_burst(L, gl, a, M, win, m, n, phase):
    """A real windowed cosine burst centred at sample n*a with frequency m/M.

    Generator-side construction (independent of oracle/ and the CUDA path):
    Re(e^{i phase} * w(t) e^{i 2 pi m t / M}) at offsets t = -gl/2 .. gl/2-1,
    circular in the signal, normalised to unit energy.
    """
    t = np.arange(-(gl // 2), gl - gl // 2)
    ang = 2.0 * np.pi * t / gl
    if win == HANN:
        w = 0.5 + 0.5 * np.cos(ang)
    else:
        w = 0.42 + 0.5 * np.cos(ang) + 0.08 * np.cos(2.0 * ang)
    burst = w * np.cos(2.0 * np.pi * m * t / M + phase)
    burst /= np.sqrt(np.sum(burst * burst))
    out = np.zeros(L)
    np.add.at(out, (n * a + t) % L, burst)
    return out


def planted_c0(seed: int = 0, Ls: int = 4096) -> np.ndarray:
    """C0: 20 random unit-norm on-grid Hann(256, a=64, M=256) bursts with
    amplitudes U[0.1, 1] plus N(0, 1e-3^2) white noise (BASELINE.json configs[0])."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.zeros(Ls)
    N = Ls // 64
    for _ in range(20):
        n = int(rng.integers(0, N))
        m = int(rng.integers(1, 128))
        ph = float(rng.uniform(0.0, 2.0 * np.pi))
        A = float(rng.uniform(0.1, 1.0))
        x += A * _planted_burst(Ls, 256, 64, 256, HANN, m, n, ph)
    x += rng.normal(0.0, 1e-3, Ls)
    return x


def planted_c1(seed: int = 1, Ls: int = 65536) -> np.ndarray:
    """C1: 200 unit-norm on-grid Blackman bursts of mixed widths 512/1024/2048
    (a = w/4, M = w), amplitudes U[0.1,1], plus white noise at -40 dB of the
    burst-sum energy (BASELINE.json configs[1])."""
    rng = np.random.Generator(np.random.PCG64(seed))
    x = np.zeros(Ls)
    widths = (512, 1024, 2048)
    for _ in range(200):
        w = widths[int(rng.integers(0, 3))]
        a, M = w // 4, w
        n = int(rng.integers(0, Ls // a))
        m = int(rng.integers(1, M // 2))
        ph = float(rng.uniform(0.0, 2.0 * np.pi))
        A = float(rng.uniform(0.1, 1.0))
        x += A * _planted_burst(Ls, w, a, M, BLACKMAN, m, n, ph)
    e = np.sum(x * x)
    noise = rng.normal(0.0, 1.0, Ls)
    noise *= np.sqrt(e * 1e-4 / np.sum(noise * noise))
    return x + noise


# ----------------------------------------------------------------------------
# audio-like signal (C2, C3, C4 segments)
# ----------------------------------------------------------------------------
def audio_like(seed: int = 2, Ls: int = 220500, fs: int = FS) -> np.ndarray:
    """5 s audio-like signal (BASELINE.json configs[2]).

    8 harmonic tones (f0 ~ U[80,800] Hz, 10 partials, amplitude 1/k, random
    phase, +-1% sinusoidal vibrato at f_v ~ U[4,7] Hz, onset U[0,3.5] s,
    duration U[0.5, 5-onset] s, 10 ms raised-cosine fades), 30 exponentially
    decaying clicks (white-noise bursts, decay 5 ms, cut at 50 ms, amplitude
    U[0.5,1]), pink noise at -30 dB of tones+clicks; normalised to max|x| = 1.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    t = np.arange(Ls) / fs
    dur_total = Ls / fs
    tones = np.zeros(Ls)
    for _ in range(8):
        f0 = rng.uniform(80.0, 800.0)
        fv = rng.uniform(4.0, 7.0)
        psi = rng.uniform(0.0, 2.0 * np.pi)
        onset = rng.uniform(0.0, min(3.5, dur_total - 0.5))
        dur = rng.uniform(0.5, dur_total - onset)
        phases = rng.uniform(0.0, 2.0 * np.pi, 10)
        i0 = int(round(onset * fs))
        i1 = min(Ls, int(round((onset + dur) * fs)))
        tt = t[i0:i1] - onset
        # integral of f(t) = f0 (1 + 0.01 sin(2 pi fv t + psi))
        base = tt + 0.01 * (np.cos(psi) - np.cos(2.0 * np.pi * fv * tt + psi)) / (2.0 * np.pi * fv)
        seg = np.zeros(i1 - i0)
        for k in range(1, 11):
            if k * f0 * 1.01 >= fs / 2:
                break
            seg += np.sin(2.0 * np.pi * k * f0 * base + phases[k - 1]) / k
        nf = min(int(0.010 * fs), (i1 - i0) // 2)
        if nf > 0:
            fade = 0.5 - 0.5 * np.cos(np.pi * np.arange(nf) / nf)
            seg[:nf] *= fade
            seg[len(seg) - nf:] *= fade[::-1]
        tones[i0:i1] += seg
    clicks = np.zeros(Ls)
    ncut = int(0.050 * fs)
    decay = np.exp(-np.arange(ncut) / (0.005 * fs))
    for _ in range(30):
        onset = rng.uniform(0.0, dur_total)
        amp = rng.uniform(0.5, 1.0)
        i0 = int(onset * fs)
        n = min(ncut, Ls - i0)
        clicks[i0:i0 + n] += amp * rng.normal(0.0, 1.0, n) * decay[:n]
    sig = tones + clicks
    white = rng.normal(0.0, 1.0, Ls)
    spec = np.fft.rfft(white)
    f = np.fft.rfftfreq(Ls, 1.0 / fs)
    spec[0] = 0.0
    spec[1:] /= np.sqrt(f[1:])
    pink = np.fft.irfft(spec, Ls)
    pink *= np.sqrt(np.sum(sig * sig) * 1e-3 / np.sum(pink * pink))
    x = sig + pink
    return x / np.max(np.abs(x))


def audio_tiled(seed: int = 1000, Ls: int = 1 << 22) -> np.ndarray:
    """C4: audio_like segments with fresh seeds seed, seed+1, ... concatenated and
    truncated to Ls samples (BASELINE.json configs[4])."""
    segs = []
    total = 0
    s = seed
    while total < Ls:
        seg = audio_like(s, 220500)
        segs.append(seg)
        total += seg.size
        s += 1
    return np.concatenate(segs)[:Ls]


_GENERATORS = {
    "planted_c0": planted_c0,
    "planted_c1": planted_c1,
    "audio_like": audio_like,
    "audio_tiled": audio_tiled,
}


def signal(cfg: Config | str, seed: int | None = None) -> np.ndarray:
    """The seeded fp64 input signal x (length Ls) of a config (``seed`` overrides the
    config's seed: further signals of the same workload, e.g. for batched runs)."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    return _GENERATORS[cfg.signal](cfg.seed if seed is None else seed, cfg.Ls)


def random_signal(L: int, seed: int) -> np.ndarray:
    """Plain N(0,1) signal for small test cases."""
    return np.random.Generator(np.random.PCG64(seed)).normal(0.0, 1.0, L)
