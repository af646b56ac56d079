"""Dev tool: aggregate it/s of mpgabor_run_batch per loop kernel (set_batch 0 = automatic,
1 = one selection), cluster size per signal and batch size B.

usage: python tools/batch_cluster_sweep.py [configs] [kernels] [clusters] [batches]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C1"]
kernels = [int(k) for k in sys.argv[2].split(",")] if len(sys.argv) > 2 else [0, 1]
clusters = [int(c) for c in sys.argv[3].split(",")] if len(sys.argv) > 3 else [16, 8, 4]
batches = [int(b) for b in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 9, 18, 36]
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    mp = MPGabor(cfg.dicts, cfg.thr, "f64")
    for kern in kernels:
        mp.set_batch(kern)
        for C in clusters:
            mp.set_launch(C, 0, 0, 0)
            for B in batches:
                X = torch.from_numpy(np.stack([siggen.signal(cfg, seed=cfg.seed + 100 * b) for b in range(B)])).cuda()
                mp.run_batch(X, cfg.maxit, cfg.errdb)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                outs = mp.run_batch(X, cfg.maxit, cfg.errdb)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1)
                atoms = sum(o.n for o in outs)
                multi = outs[0].rounds < outs[0].n
                print(name, "kernel", "multi" if multi else "single", "C", C, "B", B, mp.launch_info(),
                      f"{atoms / (ms * 1e-3):.0f} it/s aggregate, {ms:.1f} ms", flush=True)
    mp.close()
