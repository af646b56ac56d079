"""Dev tool: DGT analysis time per dictionary (C4 dictionaries on the C4 signal by default):
CUDA-event time of the pad/energy + DGT phase of mpgabor_run with maxit = 0, median of runs,
against the bytes the DGT must write (the residual grid)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
cfg = siggen.CONFIGS[name]
xd = torch.from_numpy(siggen.signal(cfg)).cuda()
esz = 16 if prec == "f64" else 8
tot_ms, tot_b = 0.0, 0
for d in list(cfg.dicts) + [None]:
    dicts = cfg.dicts if d is None else (d,)
    mp = MPGabor(dicts, cfg.thr, prec)
    mp.run(xd, 0, cfg.errdb, fetch=False)
    ts = []
    for _ in range(5):
        mp.run(xd, 0, cfg.errdb, fetch=False)
        ts.append(mp.last_timing()[0])
    t = float(np.median(ts))
    L = mp.layout(cfg.Ls)[0]
    b = sum((L // dd.a) * (dd.M // 2 + 1) * esz for dd in dicts)
    tag = "all" if d is None else f"gl{d.gl} a{d.a} M{d.M}"
    print(f"{name} {prec} {tag}: {t:.3f} ms, {b / 1e6:.1f} MB written, {b / (t * 1e-3) / 1e9:.0f} GB/s", flush=True)
    mp.close()
