"""Dev tool: Alg. 2 (resets) on the B200 -- time per selection including the per-pass
DGT + synthesis + subtraction, and the true residual energy reached vs Alg. 1.
Writes profiles/<tag>_resets.md."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
rows = []
for name, K, thr in (("C2", 30000, None), ("C2", 30000, 1e-2), ("C1", 10000, 1e-2)):
    cfg = siggen.CONFIGS[name]
    thr = cfg.thr if thr is None else thr
    x = siggen.signal(cfg)
    xd = torch.from_numpy(x).cuda()
    mp = MPGabor(cfg.dicts, thr, "f64")
    for every in (None, 10000, 3000, 1000):
        torch.cuda.synchronize()
        if every is None:
            mp.run(xd, K, -np.inf)
            t0 = time.perf_counter()
            out = mp.run(xd, K, -np.inf)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            passes = 1
        else:
            mp.run_reset(xd, K, -np.inf, every)
            t0 = time.perf_counter()
            out = mp.run_reset(xd, K, -np.inf, every)
            torch.cuda.synchronize()
            wall = time.perf_counter() - t0
            passes = mp.last_passes()
        # true residual energy of the approximation (synthesis of the atom list)
        y = mp.synth(out.atoms_dev, out.n, cfg.Ls).cpu().numpy()
        etrue = float(np.dot(x - y, x - y))
        rows.append((name, thr, every or "-", passes, out.n, 1e6 * wall / max(out.n, 1), out.energy[-1] / out.E0,
                     etrue / out.E0))
        print(rows[-1], flush=True)
    mp.close()
os.makedirs("profiles", exist_ok=True)
with open(f"profiles/{tag}_resets.md", "w") as f:
    f.write("# Alg. 2 (resets) on B200, fp64 (tools/bench_resets.py)\n\n")
    f.write("Wall time per selection of a whole run (host-side, incl. every pass's DGT, synthesis and "
            "subtraction); E_K/E_0 = the run's final energy value (estimate inside a pass); true = "
            "||x - y||^2/||x||^2 of the synthesised atom list.\n\n")
    f.write("| config | threshold | reset every | passes | atoms | us/atom (wall) | E_K/E_0 | true |\n|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        f.write(f"| {r[0]} | {r[1]:g} | {r[2]} | {r[3]} | {r[4]} | {r[5]:.3f} | {r[6]:.4e} | {r[7]:.4e} |\n")
