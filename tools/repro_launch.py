import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, siggen
from paper_2202_12380_b200.mpgabor import MPGabor
cfg = siggen.CONFIGS["C1"]
x = torch.from_numpy(siggen.signal(cfg)).cuda()
for launch in [(2, 128, 32, 1), (2, 512, 32, 1), (16, 128, 64, 0), (4, 256, 128, 1), (1, 512, 64, 0)]:
    mp = MPGabor(cfg.dicts, cfg.thr, "f64")
    mp.set_batch(8)
    mp.set_launch(*launch)
    try:
        out = mp.run(x, 3000, cfg.errdb)
        print(launch, mp.launch_info(), out.n, out.rounds, flush=True)
    except Exception as e:
        print(launch, "ERR", e, flush=True)
        break
