"""Write the oracle's full-length C3/C4 decompositions to tests/golden/ (CPU only).

Calls only ``oracle/`` (and the seeded input generator ``siggen``): no value in the
files comes from the CUDA path.  One file per config, fp64 oracle (SURVEY.md §8(c)
O1-O7: Alg. 1 P:356-387 with the Eq. (9) recursion P:424-434 and Alg. 3
P:978-1029), at the config's stated K (BASELINE.json configs; siggen.CONFIGS):

  index     int32[n]    global coefficient index p of every selection
  energy    float64[n+1] the E_k estimate trace (E_0 = ||x||^2)
  gaps      float32[n]   near-tie gap (s1 - s2)/s1 before every selection
  samp_k    int64[s]     sampled selections (every 16th, first/last 2048 all)
  samp_re, samp_im float64[s]  their adjusted coefficients c~ (Eq. (19))
  res_p     int64[r]     sampled coefficients of the final residual
  res_v     complex128[r] their values
  stop, n, E0, thr, maxit, errdb, Ls, x_sha256, loop_seconds

A sidecar ``<name>_f64.json`` holds the npz's SHA-256 and the run metadata; the
tests check it before trusting the file.

Usage:  python tools/make_oracle_golden.py C3 [C4 ...]
(C3 ~ a few minutes, C4 ~ 1-2 hours on one core.)
"""
from __future__ import annotations

import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import siggen  # noqa: E402
import oracle  # noqa: E402
from oracle import loop as oloop  # noqa: E402

GOLDEN = os.path.join(ROOT, "tests", "golden")


def sample_ks(n: int) -> np.ndarray:
    k = np.arange(n)
    return k[(k % 16 == 0) | (k < 2048) | (k >= n - 2048)]


def residual_points(index: np.ndarray, P: int, seed: int = 7) -> np.ndarray:
    rng = np.random.default_rng(seed)
    last = index[-64:].astype(np.int64)
    pts = np.concatenate([last, last - 1, last + 1, rng.integers(0, P, 4096)])
    return np.unique(np.clip(pts, 0, P - 1))


def make(name: str) -> dict:
    cfg = siggen.CONFIGS[name]
    t0 = time.time()
    x = siggen.signal(cfg)
    S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
    t1 = time.time()
    r = oloop.mp_run(S, cfg.maxit, cfg.errdb)
    t2 = time.time()
    ks = sample_ks(r.n)
    pts = residual_points(r.index, S.lay.P)
    out = dict(
        index=r.index.astype(np.int32), energy=r.energy, gaps=r.gaps.astype(np.float32),
        samp_k=ks, samp_re=r.atoms["re"][ks], samp_im=r.atoms["im"][ks],
        res_p=pts, res_v=r.res[pts],
        stop=np.int32(r.stop), n=np.int64(r.n), E0=np.float64(S.E0), thr=np.float64(cfg.thr),
        maxit=np.int64(cfg.maxit), errdb=np.float64(cfg.errdb), Ls=np.int64(cfg.Ls),
    )
    path = os.path.join(GOLDEN, f"{name}_f64.npz")
    np.savez_compressed(path, **out)
    sha = hashlib.sha256(open(path, "rb").read()).hexdigest()
    meta = dict(config=name, precision="f64", generator="siggen v1", n=int(r.n),
                stop=oloop.STOP_NAMES[r.stop], E0=float(S.E0), E_final=float(r.energy[-1]),
                min_gap=float(r.gaps.min()) if r.n else None,
                first_near_tie=int(np.argmax(r.gaps < 1e-6)) if (r.gaps < 1e-6).any() else None,
                x_sha256=hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
                npz_sha256=sha, setup_seconds=round(t1 - t0, 1), loop_seconds=round(t2 - t1, 1),
                loop_it_per_s=round(r.n / (t2 - t1), 1),
                script="tools/make_oracle_golden.py (calls oracle/ only)")
    with open(os.path.join(GOLDEN, f"{name}_f64.json"), "w") as f:
        json.dump(meta, f, indent=1)
        f.write("\n")
    return meta


if __name__ == "__main__":
    for nm in sys.argv[1:] or ["C3", "C4"]:
        print(json.dumps(make(nm)), flush=True)
