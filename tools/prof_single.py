import os, sys
sys.path.insert(0, "/root/repo")
import torch, siggen
from paper_2202_12380_b200.mpgabor import MPGabor
PH = ["wait", "select", "bar1", "update", "bar2", "lvl1", "root"]
for name, K in (("C2", 20000), ("C3", 20000), ("C4", 20000)):
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, "f64")
    mp.set_batch(1)
    mp.set_profile(1)
    mp.run(xd, K, cfg.errdb, fetch=False)
    res, _ = mp.run(xd, K, cfg.errdb, fetch=False)
    c = mp.last_profile()
    n = c[7]
    print(name, mp.launch_info(), " ".join(f"{p}={x / n:.0f}" for p, x in zip(PH, c[:7])), f"total={sum(c[:7]) / n:.0f} cycles/it", flush=True)
    mp.close()
