import sys, os
sys.path.insert(0, "/root/repo")
import torch, siggen
from paper_2202_12380_b200.mpgabor import MPGabor
cfg = siggen.CONFIGS["C2"]
xd = torch.from_numpy(siggen.signal(cfg)).cuda()
for prec in ("f64",):
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    for b in (1, 8):
        for tw in (32, 64, 128):
            mp.set_batch(b); mp.set_launch(0, 0, tw, 0)
            mp.run(xd, 100000, cfg.errdb, fetch=False)
            res, _ = mp.run(xd, 100000, cfg.errdb, fetch=False)
            loop = mp.last_timing()[2]
            print(f"{prec} batch={b} TW={tw} {mp.launch_info()} atoms {res.n_atoms} rounds {res.rounds} loop {loop:.2f} ms {1e3*loop/res.n_atoms:.3f} us/atom {1e3*loop/res.rounds:.2f} us/round", flush=True)
