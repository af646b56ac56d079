python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
import siggen
from paper_2202_12380_b200.mpgabor import MPGabor
for name in ("C1", "C2"):
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, "f64")
    for TW in (64, 32, 128):
        for b in (8, 1):
            mp.set_batch(b); mp.set_launch(0, 512, TW, 0)
            mp.run(xd, cfg.maxit, cfg.errdb, fetch=False)
            ts = []
            for _ in range(3):
                r, _ = mp.run(xd, cfg.maxit, cfg.errdb, fetch=False); ts.append(mp.last_timing()[2])
            print(name, "TW", TW, "batch", b, mp.launch_info(), f"{1e3 * min(ts) / r.n_atoms:.3f} us/atom", flush=True)
    mp.close()
PY
