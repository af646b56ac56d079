import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, siggen
from paper_2202_12380_b200.mpgabor import MPGabor
for name in ("C1", "C2", "C3"):
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, "f64")
    K = min(cfg.maxit, 30000)
    for ped in (0, 1):
        mp.set_pedantic(ped)
        mp.run(xd, K, cfg.errdb)
        out = mp.run(xd, K, cfg.errdb)
        loop = mp.last_timing()[2]
        y = mp.synth(out.atoms_dev, out.n, cfg.Ls).cpu().numpy(); x = xd.cpu().numpy()
        print(f"{name} pedantic={ped} {mp.launch_info()['cluster']}: n={out.n} {1e3*loop/out.n:.3f} us/atom, final est {out.energy[-1]/out.E0:.4e}, true {np.dot(x-y,x-y)/out.E0:.4e}", flush=True)
    mp.close()
