"""Dev tool: loop time per tile width / record placement / cluster for a config (one-selection kernel)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
prec = sys.argv[3] if len(sys.argv) > 3 else "f64"
batch = int(sys.argv[4]) if len(sys.argv) > 4 else 1
cfg = siggen.CONFIGS[name]
xd = torch.from_numpy(siggen.signal(cfg)).cuda()
mp = MPGabor(cfg.dicts, cfg.thr, prec)
mp.set_batch(batch)
for C in (16, 8):
    for tw in (32, 64, 128):
        for rec in (1, 2):
            try:
                mp.set_launch(C, 0, tw, rec)
                mp.run(xd, K, cfg.errdb, fetch=False)
                res, _ = mp.run(xd, K, cfg.errdb, fetch=False)
                loop = mp.last_timing()[2]
                print(f"{name} {prec} C={C} TW={tw} rec={'smem' if rec == 1 else 'global'}: "
                      f"{1e3 * loop / res.n_atoms:.3f} us/atom", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{name} {prec} C={C} TW={tw} rec={rec}: {e}", flush=True)
