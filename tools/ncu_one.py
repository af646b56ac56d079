"""Dev tool: one warm-up and one measured decomposition of a config (the target of an
`ncu --set full -k regex:mp_multi -s 1 -c 1` capture).  usage: python tools/ncu_one.py C2 f64 [maxit]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
cfg = siggen.CONFIGS[name]
maxit = int(sys.argv[3]) if len(sys.argv) > 3 else cfg.maxit
xd = torch.from_numpy(siggen.signal(cfg)).cuda()
mp = MPGabor(cfg.dicts, cfg.thr, prec)
for _ in range(2):
    res, _ = mp.run(xd, maxit, cfg.errdb, fetch=False)
torch.cuda.synchronize()
print(name, prec, res.n_atoms, res.rounds, mp.last_timing(), mp.launch_info())
mp.close()
