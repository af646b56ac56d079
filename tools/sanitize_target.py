"""Short runs of every loop-kernel variant for compute-sanitizer (memcheck / racecheck /
synccheck, one tool per call): C0 and C1 through the one-selection and the
multi-selection kernel, as a 16-CTA cluster and as a cooperative grid of 32 CTAs, the
candidate-list / tree / scan top-K modes, batched signals, resets and synthesis.
Prints one line per case; exits non-zero on any library error."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

K = int(sys.argv[1]) if len(sys.argv) > 1 else 300
cases = [("C0", 1, None, None), ("C0", 8, None, None), ("C1", 1, None, None), ("C1", 8, None, None),
         ("C1", 8, (32, 0, 0, 0), None), ("C1", 1, (32, 0, 0, 0), None), ("C1", 8, None, "0"),
         ("C1", 8, None, "1"), ("C1", 8, (32, 0, 0, 2), None)]
for name, batch, launch, topk in cases:
    if topk is not None:
        os.environ["MPGABOR_TOPK"] = topk
    else:
        os.environ.pop("MPGABOR_TOPK", None)
    cfg = siggen.CONFIGS[name]
    x = siggen.signal(cfg)
    mp = MPGabor(cfg.dicts, cfg.thr, "f64")
    mp.set_batch(batch)
    if launch:
        mp.set_launch(*launch)
    out = mp.run(torch.from_numpy(x).cuda(), K, cfg.errdb)
    y = mp.synth(out.atoms_dev, out.n, cfg.Ls)
    torch.cuda.synchronize()
    print(name, "batch", batch, "launch", launch, "topk", topk, "atoms", out.n, "rounds", out.rounds,
          mp.launch_info(), flush=True)
    mp.close()
cfg = siggen.CONFIGS["C1"]
X = np.stack([siggen.signal(cfg, seed=cfg.seed + 100 * b) for b in range(3)])
mp = MPGabor(cfg.dicts, cfg.thr, "f64")
outs = mp.run_batch(torch.from_numpy(X).cuda(), K, cfg.errdb)
print("batch of 3:", [o.n for o in outs], flush=True)
out = mp.run_reset(torch.from_numpy(X[0]).cuda(), K, cfg.errdb, K // 3)
print("reset:", out.n, mp.last_passes(), flush=True)
mp.close()
print("SANITIZE_TARGET_OK")
