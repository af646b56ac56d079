"""The committed full-length oracle decompositions (tests/golden/{C3,C4}_f64.npz) are
what the oracle computes today: intact (SHA-256), made from the seeded signal, and
reproduced bit for bit by a fresh oracle run over a prefix (no GPU).  Written by
tools/make_oracle_golden.py, which calls oracle/ only."""
import hashlib
import json
import os

import numpy as np
import pytest

import siggen
import oracle
from oracle import loop as oloop

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _load(name):
    path = os.path.join(GOLDEN, f"{name}_f64.npz")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated yet")
    with open(path[:-4] + ".json") as f:
        meta = json.load(f)
    with open(path, "rb") as f:
        assert hashlib.sha256(f.read()).hexdigest() == meta["npz_sha256"]
    return meta, dict(np.load(path))


@pytest.mark.parametrize("name,prefix", [("C3", 1500), ("C4", 300)])
def test_golden_is_the_oracle(name, prefix):
    meta, z = _load(name)
    cfg = siggen.CONFIGS[name]
    x = siggen.signal(cfg)
    assert hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest() == meta["x_sha256"]
    n = int(z["n"])
    assert z["index"].size == n and z["energy"].size == n + 1 and z["gaps"].size == n
    assert n == (cfg.maxit if meta["stop"] == "maxit" else n) and n <= cfg.maxit
    assert np.all(np.diff(z["energy"]) <= 0)                 # E~ >= 0 (Eq. (20) for |rho| < 1)
    assert np.all(z["gaps"] >= 0) and np.all(z["gaps"] <= 1)
    S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
    assert z["energy"][0] == S.E0
    r = oloop.mp_run(S, prefix, cfg.errdb)
    assert np.array_equal(r.index, z["index"][:prefix].astype(np.int64))
    assert np.array_equal(r.energy, z["energy"][: prefix + 1])
    assert np.array_equal(r.gaps.astype(np.float32), z["gaps"][:prefix])
    ks = z["samp_k"][z["samp_k"] < prefix]
    assert np.array_equal(r.atoms["re"][ks], z["samp_re"][: ks.size])
