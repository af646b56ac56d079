"""Dev tool: loop time of the one-selection and multi-selection kernels on several configs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3", "C4"]
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 20000
prec = sys.argv[3] if len(sys.argv) > 3 else "f64"
batches = [int(b) for b in sys.argv[4].split(",")] if len(sys.argv) > 4 else [1, 8]
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    K = min(cfg.maxit, kmax)
    ref = None
    for b in batches:
        mp.set_batch(b)
        out = mp.run(xd, K, cfg.errdb)
        out = mp.run(xd, K, cfg.errdb)
        loop = mp.last_timing()[2]
        info = mp.launch_info()
        same = "" if ref is None else (" identical" if (out.atoms.tobytes() == ref.atoms.tobytes()) else " DIFFERENT")
        ref = ref or out
        print(f"{name} {prec} batch={b} {info}: n={out.n} rounds={out.rounds} loop {loop:.1f} ms "
              f"{1e3 * loop / out.n:.3f} us/atom {out.n / (loop * 1e-3):.0f} it/s{same}", flush=True)
    mp.close()
