"""Dev tool: A/B timing of library builds / launch settings on full decompositions.

usage: MPGABOR_LIB=<lib.so> python tools/ab_run.py <tag> <configs> <prec> <runs> [cluster threads tw rec] [batch]
Prints one line per config: loop us/atom (median of runs), atoms, rounds, launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

tag = sys.argv[1]
cfgs = sys.argv[2].split(",")
prec = sys.argv[3]
runs = int(sys.argv[4])
launch = tuple(int(v) for v in sys.argv[5].split(",")) if len(sys.argv) > 5 and sys.argv[5] != "-" else None
batch = int(sys.argv[6]) if len(sys.argv) > 6 else None
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    if launch:
        mp.set_launch(*launch)
    if batch is not None:
        mp.set_batch(batch)
    bufs = mp.alloc(cfg.maxit, cfg.Ls)
    mp.run(xd, cfg.maxit, cfg.errdb, bufs=bufs, fetch=False)
    ts = []
    for _ in range(runs):
        res, _ = mp.run(xd, cfg.maxit, cfg.errdb, bufs=bufs, fetch=False)
        ts.append(mp.last_timing()[2])
    t = float(np.median(ts))
    print(f"{tag} {name} {prec}: {1e3 * t / res.n_atoms:.4f} us/atom ({res.n_atoms / (t * 1e-3):.0f} it/s) "
          f"atoms {res.n_atoms} rounds {res.rounds} loop {t:.2f} ms [{min(ts):.2f}..{max(ts):.2f}] "
          f"{mp.launch_info()}", flush=True)
    mp.close()
