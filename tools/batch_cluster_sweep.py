import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, siggen
from paper_2202_12380_b200.mpgabor import MPGabor
for name in ("C2", "C1"):
    cfg = siggen.CONFIGS[name]
    mp = MPGabor(cfg.dicts, cfg.thr, "f64")
    for C in (16, 8, 4):
        mp.set_launch(C, 0, 0, 0)
        for B in (1, 9, 18, 36):
            X = torch.from_numpy(np.stack([siggen.signal(cfg, seed=cfg.seed + 100 * b) for b in range(B)])).cuda()
            mp.run_batch(X, cfg.maxit, cfg.errdb)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); outs = mp.run_batch(X, cfg.maxit, cfg.errdb); e1.record(); torch.cuda.synchronize()
            ms = e0.elapsed_time(e1); atoms = sum(o.n for o in outs)
            print(name, "C", C, "B", B, mp.launch_info()["cluster"], f"{atoms / (ms * 1e-3):.0f} it/s aggregate, {ms:.1f} ms", flush=True)
    mp.close()
