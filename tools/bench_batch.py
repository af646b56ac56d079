"""Dev tool: batched independent decompositions (mpgabor_run_batch) -- aggregate MP
iterations/s over B signals of a config (one cluster each, automatic size and loop kernel), vs one signal.
Writes profiles/<tag>_batch.md."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["C2", "C1"]
rows = []
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    for prec in ("f64",):
        mp = MPGabor(cfg.dicts, cfg.thr, prec)
        for B in (1, 4, 9, 18, 36, 72):
            X = torch.from_numpy(np.stack([siggen.signal(cfg, seed=cfg.seed + 100 * b) for b in range(B)])).cuda()
            mp.run_batch(X, cfg.maxit, cfg.errdb, fetch=False)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            res, _, _ = mp.run_batch(X, cfg.maxit, cfg.errdb, fetch=False)   # synchronises; no host copies
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1)
            atoms = sum(r.n_atoms for r in res)
            kern = "multi" if res[0].rounds < res[0].n_atoms else "single"
            rows.append((name, prec, B, atoms, ms, atoms / (ms * 1e-3), mp.last_timing()[2], mp.launch_info()["cluster"], kern))
            print(rows[-1], flush=True)
        mp.close()
os.makedirs("profiles", exist_ok=True)
with open(f"profiles/{tag}_batch.md", "w") as f:
    f.write("# Batched independent signals (mpgabor_run_batch), B200\n\n")
    f.write("B signals of the config (seeds seed + 100 b), each decomposed to its stop rule by its own "
            "cluster (automatic cluster size and loop kernel: multi-selection for C1/C2); time = CUDA events "
            "around the whole C-ABI call (DGT of every signal, tile init, loop, result copy; atoms stay on the "
            "device); "
            "aggregate = total selections / time.\n\n")
    f.write("| config | prec | B | kernel | CTAs per signal | selections | ms | aggregate it/s | loop ms |\n|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        f.write(f"| {r[0]} | {r[1]} | {r[2]} | {r[8]} | {r[7]} | {r[3]} | {r[4]:.2f} | {r[5]:.0f} | {r[6]:.2f} |\n")
