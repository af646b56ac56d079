"""Dev tool: per-phase cycle breakdown of the persistent loop + launch-parameter sweep."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

PH = ["wait", "select", "bar1", "update", "bar2", "lvl1", "root"]


def one(mp, xd, K, errdb, mode):
    mp.set_profile(mode)
    out = mp.run(xd, K, errdb, fetch=False)
    res = out[0]
    c = mp.last_profile()
    dgt, init, loop = mp.last_timing()
    n = max(1, c[7])
    tot = sum(c[:7])
    ghz = tot / (loop * 1e6) if loop > 0 else 0
    per = [x / n / ghz for x in c[:7]] if ghz else [0] * 7
    return res.n_atoms, loop, ghz, per


def main():
    cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C0", "C2"]
    K = int(sys.argv[2]) if len(sys.argv) > 2 else 5000
    sweep = len(sys.argv) > 3 and sys.argv[3] == "sweep"
    for name in cfgs:
        cfg = siggen.CONFIGS[name]
        x = siggen.signal(cfg)
        xd = torch.from_numpy(x).cuda()
        for prec in ("f64", "f32"):
            mp = MPGabor(cfg.dicts, cfg.thr, prec)
            grid = [(0, 0, 0)]
            if sweep:
                grid = list(itertools.product((2, 4, 8, 16), (128, 256, 512), (32, 64, 128)))
            for (C, T, TW) in grid:
                try:
                    mp.set_launch(C, T, TW, 0)
                    one(mp, xd, K, cfg.errdb, 1)
                    info = mp.launch_info()
                    n, loop, ghz, per = one(mp, xd, K, cfg.errdb, 1)
                    nf, loopf, _, perf = one(mp, xd, K, cfg.errdb, 3)
                except Exception as e:  # noqa: BLE001
                    print(name, prec, C, T, TW, "ERR", e, flush=True)
                    continue
                us = 1e3 * loop / max(n, 1)
                usf = 1e3 * loopf / max(nf, 1)
                print(f"{name} {prec} C={info['cluster']} T={info['threads']} TW={info['tile_width']} {info['records']}: {n} it, {us:.3f} us/it ({1e6/us:.0f} it/s), "
                      f"floor {usf:.3f} us/it, clk {ghz:.2f} GHz | " +
                      " ".join(f"{p}={v*1e-3:.3f}" for p, v in zip(PH, per)) +
                      " | floor: " + " ".join(f"{v*1e-3:.3f}" for v in perf), flush=True)
            mp.close()


if __name__ == "__main__":
    main()
