import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, siggen
import paper_2202_12380_b200.mpgabor as mpg
cfg = siggen.CONFIGS["C2"]
x = torch.from_numpy(siggen.signal(cfg)).cuda()
mp = mpg.MPGabor(cfg.dicts, cfg.thr, "f64")
for kind, T, TW in ((0, 512, 64), (0, 512, 32), (4, 512, 32), (4, 256, 64)):
    mp.set_profile(kind); mp.set_launch(0, T, TW, 0)
    mp.run(x, cfg.maxit, cfg.errdb, fetch=False)
    r = mp.run(x, cfg.maxit, cfg.errdb, fetch=False)[0]
    print(kind, T, TW, mp.last_timing()[2] / r.n_atoms * 1e3, "us/it")
