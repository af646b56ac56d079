"""Dev tool: multi-selection loop vs one-selection loop vs oracle (parity + loop timing).

usage: python tools/multi_check.py C0,C1,C2 [maxit] [f64|f32] [batches, e.g. 1,4,8,0]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import oracle
import siggen
from oracle import loop as oloop
from paper_2202_12380_b200.mpgabor import MPGabor

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C0", "C1", "C2"]
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
prec = sys.argv[3] if len(sys.argv) > 3 else "f64"
batches = [int(b) for b in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 0]
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    x = siggen.signal(cfg)
    K = min(cfg.maxit, kmax)
    t = time.time()
    S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
    ref = oloop.mp_run(S, K, cfg.errdb)
    print(f"{name} {prec}: oracle n={ref.n} stop={ref.stop_name} ({time.time() - t:.1f}s)", flush=True)
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    xd = torch.from_numpy(x).cuda()
    lay = mp.layout(cfg.Ls)
    for b in batches:
        mp.set_batch(b)
        out = mp.run(xd, K, cfg.errdb)
        times = []
        for rep in range(3):
            out = mp.run(xd, K, cfg.errdb)
            times.append(mp.last_timing()[2])
        loopms = float(np.median(times))
        gi = out.index(lay[3], lay[2])
        n = min(out.n, ref.n)
        diff = np.nonzero(gi[:n] != ref.index[:n])[0]
        first = int(diff[0]) if diff.size else -1
        m = n if first < 0 else first
        rel = np.max(np.abs(out.energy[:m + 1] - ref.energy[:m + 1]) / np.abs(ref.energy[:m + 1]))
        ok = first < 0 and out.n == ref.n
        print(f"  batch={b}: n={out.n} rounds={out.rounds} ({out.n / max(out.rounds, 1):.2f} atoms/round) "
              f"stop={out.stop_name} first-diverge={first} relE={rel:.2e} {'OK' if ok else 'MISMATCH'} | "
              f"loop {loopms:.3f} ms = {loopms * 1e3 / max(out.n, 1):.3f} us/atom, {out.n / (loopms * 1e-3):.0f} it/s",
              flush=True)
    mp.close()
