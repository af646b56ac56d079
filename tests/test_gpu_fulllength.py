"""Full-length parity on C3/C4 against committed oracle decompositions, exact ties,
and synthesis of the large dictionaries (B200 only).

North_star acceptance (BASELINE.json) at the configs' stated K:
  fp64: identical atom-index sequence, |E_k^gpu - E_k^or| <= 1e-9 max(|E_k^or|, 1e-4 E_0)
        at every k (reading Z23), sampled c~ and final residual coefficients within
        1e-9 sqrt(E_0);
  fp32: identical indices up to the first oracle near-tie; a divergence before it is
        accepted only where the oracle gap is within the fp32 drift estimate of
        SURVEY.md §8(c) "numerical budget"; final estimate within 1e-4 E_0 (Z20).
        Every run writes its first divergence index, the oracle gap there and the drift
        estimate to gpurun_out/parity/ (copied to profiles/ per round).
The references are tests/golden/{C3,C4}_f64.npz, written by tools/make_oracle_golden.py
from oracle/ alone (Alg. 1, Eq. (9), Alg. 3); the test
first checks their SHA-256 and that they were made from this signal.
"""
import hashlib
import json
import math
import os

import numpy as np
import pytest
import torch

import siggen
from siggen import Dict, HANN, BLACKMAN, CONFIGS
import oracle
from oracle import gabor, loop as oloop

from test_gpu_parity import (energy_rel_error, first_divergence, setup_of, FP64_E_TOL, NEAR_TIE,  # noqa: F401
                             mpg)

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
OUTDIR = os.path.join(ROOT, "gpurun_out", "parity")

_G = {}


def golden(name):
    if name not in _G:
        path = os.path.join(GOLDEN, f"{name}_f64.npz")
        if not os.path.exists(path):
            pytest.skip(f"{path} not generated yet (tools/make_oracle_golden.py {name})")
        with open(path[:-4] + ".json") as f:
            meta = json.load(f)
        with open(path, "rb") as f:
            assert hashlib.sha256(f.read()).hexdigest() == meta["npz_sha256"], "golden file altered"
        z = dict(np.load(path))
        x, _ = setup_of(name)
        assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == meta["x_sha256"]
        _G[name] = (meta, z)
    return _G[name]


def touched_mean(S):
    """Mean coefficients an update touches (kernel boxes subsampled per target, averaged
    over the selected dictionary)."""
    W = len(S.dicts)
    tot = 0.0
    for u in range(W):
        for v in range(W):
            K = S.K[u * W + v]
            s_m = K.M_c // S.dicts[v].M
            s_n = max(1, S.dicts[v].a // K.a_c)
            tot += math.ceil(K.h.shape[0] / s_n) * math.ceil(K.h.shape[1] / s_m)
    return tot / W


def fp32_drift(S, k):
    """Score drift estimate of SURVEY.md §8(c): a coefficient has received about
    n = k * touched / P_R updates, each adding fp32 rounding of ~6e-8 relative; the score
    (|c|^2) drifts by ~2 sqrt(n) 6e-8 relative."""
    n = k * touched_mean(S) / S.lay.P
    return 2.0 * math.sqrt(max(n, 1.0)) * 6e-8


def write_report(tag, rec):
    os.makedirs(OUTDIR, exist_ok=True)
    with open(os.path.join(OUTDIR, f"{tag}.json"), "w") as f:
        json.dump(rec, f, indent=1)
        f.write("\n")


def run_full(mpg, name, prec, batch=None, launch=None, K=None):
    cfg = CONFIGS[name]
    x, S = setup_of(name)
    mp = mpg.MPGabor(cfg.dicts, cfg.thr, prec)
    if batch is not None:
        mp.set_batch(batch)
    if launch is not None:
        mp.set_launch(*launch)
    out = mp.run(torch.from_numpy(x).cuda(), cfg.maxit if K is None else K, cfg.errdb)
    lay = mp.layout(cfg.Ls)
    return mp, out, out.index(lay[3], lay[2])


# ---------------------------------------------------------------------------
# fp64: the full C3 (105k atoms, negative-estimate stop) and C4 (1e6 atoms) runs
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("batch", [0, 1])   # automatic (multi-selection on a grid), one selection
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_length_fp64_vs_oracle(mpg, name, batch):
    meta, z = golden(name)
    x, S = setup_of(name)
    mp, out, idx = run_full(mpg, name, "f64", batch=batch)
    ref_idx = z["index"].astype(np.int64)
    d = first_divergence(idx, ref_idx)
    rel = energy_rel_error(out.energy[: d + 1], z["energy"][: d + 1], S.E0)
    write_report(f"{name}_f64_b{batch}", dict(config=name, precision="f64", kernel_batch=batch, n_gpu=int(out.n),
                                              n_oracle=int(z["n"]), first_divergence=d,
                                              stop_gpu=out.stop_name, stop_oracle=meta["stop"],
                                              max_rel_energy_error=float(rel.max()),
                                              cluster=mp.launch_info()["cluster"], rounds=int(out.rounds)))
    assert out.n == int(z["n"]) and out.stop == int(z["stop"]), (out.n, int(z["n"]), out.stop_name, meta["stop"])
    assert np.array_equal(idx, ref_idx), f"first divergence at {d}"
    assert rel.max() <= FP64_E_TOL, rel.max()
    ks = z["samp_k"]
    tol = 1e-9 * math.sqrt(S.E0)
    assert np.max(np.abs(out.atoms["re"][ks] - z["samp_re"])) <= tol
    assert np.max(np.abs(out.atoms["im"][ks] - z["samp_im"])) <= tol
    res = mp.residual(CONFIGS[name].Ls).cpu().numpy()
    assert np.max(np.abs(res[z["res_p"]] - z["res_v"])) <= tol
    mp.close()


# ---------------------------------------------------------------------------
# fp32 at full length: first divergence, the oracle gap there, the drift estimate
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_full_length_fp32_vs_oracle(mpg, name):
    meta, z = golden(name)
    x, S = setup_of(name)
    mp, out, idx = run_full(mpg, name, "f32")
    ref_idx = z["index"].astype(np.int64)
    gaps = z["gaps"].astype(np.float64)
    n = min(out.n, ref_idx.size)
    d = first_divergence(idx, ref_idx)
    diverged = d < n
    first_tie = int(np.argmax(gaps < NEAR_TIE)) if (gaps < NEAR_TIE).any() else None
    drift = fp32_drift(S, d)
    dE = abs(out.energy[-1] - z["energy"][-1]) / S.E0
    rec = dict(config=name, precision="f32", n_gpu=int(out.n), n_oracle=int(z["n"]), stop_gpu=out.stop_name,
               stop_oracle=meta["stop"], first_divergence=d if diverged else None,
               oracle_gap_at_divergence=float(gaps[d]) if diverged else None,
               min_oracle_gap_up_to_divergence=float(gaps[: d + 1].min()) if diverged else None,
               first_oracle_near_tie=first_tie, drift_estimate_at_divergence=drift,
               final_energy_error_rel_E0=dE, cluster=mp.launch_info()["cluster"])
    write_report(f"{name}_f32", rec)
    if diverged:
        # allowed at or after an oracle near-tie, or where the gap is within the drift
        assert gaps[: d + 1].min() < max(NEAR_TIE, 10.0 * drift), rec
    assert dE <= 1e-4, rec
    mp.close()


# ---------------------------------------------------------------------------
# exact ties (reading Z10: the lowest global index wins) through every loop variant
# ---------------------------------------------------------------------------
def _twin_burst_signal():
    # one windowed burst copied bit for bit to frames 4 and 20 of a 16/4/16 Hann
    # dictionary: both frames hold identical samples, so their DGT values tie exactly
    d = Dict(HANN, 16, 4, 16)
    L = 128
    j = np.arange(-8, 8)
    burst = (0.5 + 0.5 * np.cos(2 * np.pi * j / 16)) * np.cos(2 * np.pi * 3 * j / 16 + 0.3)
    x = np.zeros(L)
    x[4 * 4 + j] = burst
    x[20 * 4 + j] = burst
    return (d,), x


def _periodic_signal():
    # period 64 samples (a multiple of every hop) dividing L = 1024: every frame of a
    # dictionary repeats exactly every 64/a frames -> families of exact ties at every step
    dicts = (Dict(BLACKMAN, 32, 8, 32), Dict(HANN, 64, 16, 64))
    rng = np.random.Generator(np.random.PCG64(5))
    x = np.tile(rng.standard_normal(64), 16)
    return dicts, x


TIE_VARIANTS = [("batch1", 1, None), ("auto", 0, None), ("batch8", 8, None), ("grid32", 8, (32, 0, 0, 0)),
                ("grid64", 8, (64, 0, 0, 0)), ("grid128", 8, (128, 0, 0, 0)), ("single_grid32", 1, (32, 0, 0, 0))]


@pytest.mark.parametrize("variant,batch,launch", TIE_VARIANTS)
@pytest.mark.parametrize("case", ["twin", "periodic"])
def test_exact_ties(mpg, case, variant, batch, launch):
    dicts, x = _twin_burst_signal() if case == "twin" else _periodic_signal()
    thr, K = 1e-4, (2 if case == "twin" else 120)
    S = oracle.Setup.build(x, dicts, thr)
    ref = oloop.mp_run(S, K, -60.0)
    if case == "twin":
        s = np.abs(S.grids[0]) ** 2
        assert s[4, 3] == s[20, 3] and ref.gaps[0] == 0.0
        assert (ref.atoms["n"][0], ref.atoms["m"][0]) == (4, 3)
    else:
        assert (ref.gaps[:K] == 0.0).sum() >= 10      # many exact ties along the way
    mp = mpg.MPGabor(dicts, thr, "f64")
    mp.set_batch(batch)
    if launch is not None:
        mp.set_launch(*launch)
    out = mp.run(torch.from_numpy(x).cuda(), K, -60.0)
    lay = mp.layout(x.size)
    idx = out.index(lay[3], lay[2])
    assert out.n == ref.n and np.array_equal(idx, ref.index), first_divergence(idx, ref.index)
    assert energy_rel_error(out.energy, ref.energy, ref.energy[0]).max() <= FP64_E_TOL
    mp.close()


@pytest.mark.parametrize("kernel", [0, 1])
def test_exact_ties_batched(mpg, kernel):
    dicts, x = _periodic_signal()
    S = oracle.Setup.build(x, dicts, 1e-4)
    ref = oloop.mp_run(S, 120, -60.0)
    X = np.stack([x, np.roll(x, 8), x])
    mp = mpg.MPGabor(dicts, 1e-4, "f64")
    mp.set_batch(kernel)
    outs = mp.run_batch(torch.from_numpy(X).cuda(), 120, -60.0)
    lay = mp.layout(x.size)
    for b in (0, 2):
        assert np.array_equal(outs[b].index(lay[3], lay[2]), ref.index), b
    assert outs[0].atoms.tobytes() == outs[2].atoms.tobytes()
    mp.close()


# ---------------------------------------------------------------------------
# synthesis (Eq. (18)) with the C3 / C4 dictionary shapes, and its determinism
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["C3", "C4"])
def test_synthesis_large_dictionaries(mpg, name):
    cfg = CONFIGS[name]
    x, S = setup_of(name)
    mp, out, _ = run_full(mpg, name, "f64", K=4000)
    y = mp.synth(out.atoms_dev, out.n, cfg.Ls).cpu().numpy()
    yref = gabor.synthesize(out.atoms, cfg.dicts, S.lay.L, cfg.Ls)
    assert np.max(np.abs(y - yref)) <= 1e-11 * np.max(np.abs(yref))
    mp.close()


def test_synthesis_deterministic_with_repeated_atoms(mpg):
    # the same coefficient selected many times: sol(p) sums in atom-list order (Z19),
    # bit for bit on every call, and equals the oracle's Eq. (18)
    cfg = CONFIGS["C1"]
    x, S = setup_of("C1")
    mp, out, _ = run_full(mpg, "C1", "f64", K=3000)
    rng = np.random.default_rng(3)
    at = out.atoms
    rep = np.concatenate([at, at[rng.integers(0, 50, 2000)], at[::-1][:500]])
    rep["re"] *= rng.uniform(0.5, 1.5, rep.size)
    dev = torch.from_numpy(rep.view(np.uint8).copy()).cuda()
    y1 = mp.synth(dev, rep.size, cfg.Ls).cpu().numpy()
    y2 = mp.synth(dev, rep.size, cfg.Ls).cpu().numpy()
    assert y1.tobytes() == y2.tobytes()
    yref = gabor.synthesize(rep, cfg.dicts, S.lay.L, cfg.Ls)
    assert np.max(np.abs(y1 - yref)) <= 1e-11 * np.max(np.abs(yref))
    mp.close()
