"""Dev tool: a short, fixed run for ncu captures (C2 fp64 by default)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
prec = sys.argv[3] if len(sys.argv) > 3 else "f64"
cfg = siggen.CONFIGS[name]
x = torch.from_numpy(siggen.signal(cfg)).cuda()
mp = MPGabor(cfg.dicts, cfg.thr, prec)
for _ in range(2):
    out = mp.run(x, K, cfg.errdb, fetch=False)
torch.cuda.synchronize()
print(name, prec, "done", out[0].n_atoms, mp.launch_info(), mp.last_timing())
