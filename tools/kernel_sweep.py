"""Dev tool: loop time of each loop kernel / thread count / tile width on a config (parity checked)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
import paper_2202_12380_b200.mpgabor as mpg

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    x = torch.from_numpy(siggen.signal(cfg)).cuda()
    for prec in ("f64", "f32"):
        mp = mpg.MPGabor(cfg.dicts, cfg.thr, prec)
        ref = None
        res = []
        for kind, kname in ((0, "lean"), (4, "legacy"), (8, "flat")):
            for T in ((128, 256, 512) if kind != 8 else (0,)):
                for TW in (32, 64, 128):
                    try:
                        mp.set_profile(kind)
                        mp.set_launch(0, T, TW, 0)
                        out = mp.run(x, min(K, cfg.maxit), cfg.errdb)
                        out = mp.run(x, min(K, cfg.maxit), cfg.errdb)
                        lay = mp.layout(cfg.Ls)
                        idx = out.index(lay[3], lay[2])
                        if ref is None:
                            ref = idx
                        same = np.array_equal(idx, ref) if prec == "f64" else None
                        loop = mp.last_timing()[2]
                        info = mp.launch_info()
                        res.append((loop / out.n * 1e3, kname, info["threads"], info["tile_width"], info["records"],
                                    info["cluster"], same, out.n))
                    except Exception as e:  # noqa: BLE001
                        print(name, prec, kname, T, TW, "ERR", e)
        for r in sorted(res)[:8]:
            print(f"{name} {prec} {r[0]:.3f} us/it ({1e6 / r[0]:.0f} it/s) kernel={r[1]} T={r[2]} TW={r[3]} {r[4]} "
                  f"C={r[5]} same_seq={r[6]} n={r[7]}", flush=True)
        mp.close()
