"""Ad-hoc GPU check: parity vs oracle + timings for a few configs (dev tool)."""
import sys, time, os, math
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import siggen, oracle
from oracle import loop as oloop, gabor
from paper_2202_12380_b200.mpgabor import MPGabor

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C0", "C1", "C2"]
kmax = int(sys.argv[2]) if len(sys.argv) > 2 else 10**9
prec = sys.argv[3] if len(sys.argv) > 3 else "f64"
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    x = siggen.signal(cfg)
    K = min(cfg.maxit, kmax)
    t = time.time()
    S = oracle.Setup.build(x, cfg.dicts, cfg.thr)
    ref = oloop.mp_run(S, K, cfg.errdb)
    tor = time.time() - t
    t = time.time()
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    torch.cuda.synchronize()
    tk = time.time() - t
    print(name, prec, "kernel stats", mp.kernel_stats(), "oracle entries", sum(k.h.size for k in S.K), "kept", sum(k.kept for k in S.K), flush=True)
    # kernel parity
    W = len(cfg.dicts)
    kerr = 0.0; boxok = True
    for u in range(W):
        for v in range(W):
            box, vals, mx = mp.kernel_box(u, v)
            K0 = S.K[u * W + v]
            if box != (K0.mu_lo, K0.mu_hi, K0.nu_lo, K0.nu_hi) or not np.array_equal(vals != 0, K0.h != 0):
                boxok = False
                print("  box mismatch", u, v, box, (K0.mu_lo, K0.mu_hi, K0.nu_lo, K0.nu_hi))
            else:
                kerr = max(kerr, np.max(np.abs(vals - K0.h)))
    print("  kernels: boxes/kept identical", boxok, "max abs err", kerr, flush=True)
    xd = torch.from_numpy(x).cuda()
    out = mp.run(xd, K, cfg.errdb)
    for rep in range(2):
        t0 = time.time(); out = mp.run(xd, K, cfg.errdb); t1 = time.time()
    dgt, init, loopms = mp.last_timing()
    lay = mp.layout(cfg.Ls)
    gi = out.index(lay[3], lay[2])
    n = min(out.n, ref.n)
    same = np.nonzero(gi[:n] != ref.index[:n])[0]
    first = int(same[0]) if same.size else -1
    m = n if first < 0 else first
    rel = np.max(np.abs(out.energy[:m + 1] - ref.energy[:m + 1]) / np.abs(ref.energy[:m + 1]))
    print(f"  gpu n={out.n} stop={out.stop_name} cluster={out.cluster} | oracle n={ref.n} stop={ref.stop_name} | first diverge {first} (gap there {ref.gaps[first] if first>=0 else None}) | max rel E err {rel:.3e}", flush=True)
    print(f"  timing: wall {1e3*(t1-t0):.2f} ms; dgt {dgt:.3f} ms init {init:.3f} ms loop {loopms:.3f} ms -> {out.n/(loopms*1e-3):.0f} it/s loop-only; oracle {tor:.2f}s ({ref.n/tor:.0f} it/s incl setup)", flush=True)
    y = mp.synth(out.atoms_dev, out.n, cfg.Ls).cpu().numpy()
    yref = gabor.synthesize(ref.atoms[:m], cfg.dicts, S.lay.L, cfg.Ls) if first >= 0 else gabor.synthesize(ref.atoms, cfg.dicts, S.lay.L, cfg.Ls)
    if first < 0:
        print("  synth max abs err", np.max(np.abs(y - yref)), "rel", np.max(np.abs(y-yref))/np.max(np.abs(yref)), flush=True)
    mp.close()
