"""Dev tool: loop time per atom over tile width, record placement and loop kernel.

usage: python tools/tw_sweep.py [configs] [maxit] [precision] [batches] [tws] [records]
records: 0 automatic, 1 shared, 2 global (mpgabor_set_launch)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor, MpgError

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3", "C4"]
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
prec = sys.argv[3] if len(sys.argv) > 3 else "f64"
batches = [int(b) for b in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 8]
tws = [int(t) for t in sys.argv[5].split(",")] if len(sys.argv) > 5 else [32, 64, 128]
recs = [int(r) for r in sys.argv[6].split(",")] if len(sys.argv) > 6 else [0, 2]
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    K = min(cfg.maxit, kmax)
    for b in batches:
        for tw in tws:
            for rc in recs:
                mp.set_batch(b)
                mp.set_launch(0, 512, tw, rc)
                try:
                    mp.run(xd, K, cfg.errdb, fetch=False)
                    r, _ = mp.run(xd, K, cfg.errdb, fetch=False)
                except MpgError as e:
                    print(name, prec, "batch", b, "TW", tw, "rec", rc, "->", e, flush=True)
                    continue
                lm = mp.last_timing()[2]
                print(name, prec, "batch", b, "TW", tw, "rec", rc, mp.launch_info(),
                      f"{1e3 * lm / r.n_atoms:.3f} us/atom", flush=True)
    mp.close()
