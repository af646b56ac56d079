"""Dev tool: how many consecutive MP selections are mutually independent at tile granularity.

Runs the oracle on a config, then for every selection computes the (superset of the) set of
tiles (dictionary v, frame, TW-bin tile) its update touches and simulates the speculative
multi-selection round of mpmulti.cu: a round starts at selection i and accepts i+1, i+2, ...
while the next selection's tile is outside the union of the round's touched tiles
(and at most KMAX per round).  Prints the mean accepted atoms per round.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import siggen
from oracle import gabor, loop

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
TW = int(sys.argv[2]) if len(sys.argv) > 2 else 64
cfg = siggen.CONFIGS[name]
x = siggen.signal(cfg)
S = gabor.Setup.build(x, cfg.dicts, cfg.thr)
r = loop.mp_run(S, cfg.maxit, cfg.errdb, want_gaps=False)
lay = S.lay
W = len(cfg.dicts)
print(name, "atoms", r.n)


def touched(w, m, n):
    du = cfg.dicts[w]
    out = set()
    for v in range(W):
        K = S.K[w * W + v]
        dv = cfg.dicts[v]
        a_c, M_c = K.a_c, K.M_c
        t0 = n * du.a
        f_lo = -((-(t0 + K.nu_lo * a_c)) // dv.a)
        f_hi = (t0 + K.nu_hi * a_c) // dv.a
        kp = m * (M_c // du.M)
        sm = M_c // dv.M
        q_lo = -((-(kp + K.mu_lo)) // sm)
        q_hi = (kp + K.mu_hi) // sm
        bins = set()
        for q in range(q_lo, q_hi + 1):
            qq = q % dv.M
            bins.add(min(qq, dv.M - qq))
        tiles = {b // TW for b in bins}
        for f in range(f_lo, f_hi + 1):
            for t in tiles:
                out.add((v, f % lay.N[v], t))
    return out


at = r.atoms
tiles = [(int(a["w"]), int(a["n"]) , int(a["m"]) // TW) for a in at]
T = [touched(int(a["w"]), int(a["m"]), int(a["n"])) for a in at]
for KMAX in (4, 8, 16, 64):
    rounds, i, fails = 0, 0, 0
    while i < r.n:
        U = set(T[i])
        j = i + 1
        while j < r.n and j - i < KMAX and tiles[j] not in U:
            U |= T[j]
            j += 1
        if j < r.n and j - i < KMAX:
            fails += 1
        rounds += 1
        i = j
    print(f"KMAX={KMAX}: rounds {rounds}, atoms/round {r.n / rounds:.2f}, rounds ending in a dependency {fails}")
print("mean touched tiles per atom", np.mean([len(t) for t in T[:2000]]))
