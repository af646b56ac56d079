"""Dev tool: the one-selection loop as a cooperative grid (global root exchange) vs one cluster."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2", "C3", "C4"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
prec = sys.argv[3] if len(sys.argv) > 3 else "f64"
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    mp.set_batch(1)
    ref = None
    for C in (16, 32, 64, 128):
        for tw in (0, 64, 128):
            try:
                mp.set_launch(C, 0, tw, 0)
                out = mp.run(xd, K, cfg.errdb)
                out = mp.run(xd, K, cfg.errdb)
                loop = mp.last_timing()[2]
                same = "" if ref is None else (" identical" if out.atoms.tobytes() == ref.atoms.tobytes() else " DIFFERENT")
                ref = ref or out
                print(f"{name} {prec} C={C} {mp.launch_info()}: {1e3 * loop / out.n:.3f} us/atom{same}", flush=True)
            except Exception as e:  # noqa: BLE001
                print(f"{name} {prec} C={C} TW={tw}: {e}", flush=True)
    mp.close()
