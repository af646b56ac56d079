import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, siggen
from paper_2202_12380_b200.mpgabor import MPGabor
def run(name, tw, K, prec="f64"):
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    outs = {}
    for b in (1, 8):
        mp.set_batch(b); mp.set_launch(0, 0, tw, 0)
        outs[b] = mp.run(xd, K, cfg.errdb)
    a, c = outs[1].atoms, outs[8].atoms
    n = min(len(a), len(c))
    bad = [i for i in range(n) if a[i].tobytes() != c[i].tobytes()]
    print(name, "TW", tw, mp.launch_info(), "n", len(a), len(c), "first diff", bad[:1], flush=True)
    if bad:
        i = bad[0]
        print("  single", a[i - 1:i + 2]); print("  multi ", c[i - 1:i + 2])
    mp.close()
run("C2", 128, 20000)
run("C3", 64, 20000)
run("C3", 128, 20000)
run("C3", 32, 20000)
