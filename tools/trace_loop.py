"""Dev tool: per-iteration event timeline of the persistent loop (SM clock64 cycles).

Every event is taken relative to the same CTA's "roots received" event (slot 0) of
that iteration; cross-iteration latency = next iteration's slot 0 minus this one.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import siggen
import paper_2202_12380_b200.mpgabor as mpg

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
prec = sys.argv[2] if len(sys.argv) > 2 else "f64"
launch = tuple(int(v) for v in sys.argv[3].split(",")) if len(sys.argv) > 3 else (0, 0, 0, 0)
mode = int(sys.argv[4]) if len(sys.argv) > 4 else 0
it0, n = 1000, 256
cfg = siggen.CONFIGS[name]
x = torch.from_numpy(siggen.signal(cfg)).cuda()
mp = mpg.MPGabor(cfg.dicts, cfg.thr, prec)
mp.set_launch(*launch)
mp.set_profile(mode)
mp.run(x, it0 + n + 10, cfg.errdb, fetch=False)
mpg.mpgabor_set_trace(mp.h, it0, n)
mp.run(x, it0 + n + 10, cfg.errdb, fetch=False)
T = mpg.mpgabor_last_trace(mp.h, n).astype(np.float64)       # [it][cta][slot]
info = mp.launch_info()
C, S = T.shape[1], T.shape[2]
NW = S - 13
names = {0: "roots recv", 1: "scalar done", 2: "w2 registered / geom", 3: "after B1", 4: "published",
         5: "items (count)", 6: "dirty (count)", 7: "after C (lean) / clean done (flat)"}
for w in range(NW):
    names[8 + w] = f"warp{w} items done"
names.update({8 + NW: "w2 decoded", 9 + NW: "w2 geometry", 10 + NW: "w2 loads issued", 11 + NW: "w2 c~ ready",
              12 + NW: "w2 first record+node"})
print(name, prec, info, "cycles rel. to roots received on the same CTA")
rel = T[:-1] - T[:-1, :, :1]
nxt = T[1:, :, 0] - T[:-1, :, 0]
print(f"  {'iteration period':28s} mean {nxt.mean():8.0f}  p50 {np.median(nxt):8.0f}  p90 {np.percentile(nxt, 90):8.0f}")
for s in range(S):
    if s in (5, 6):
        v = T[:-1, :, s]
        print(f"  {names[s]:28s} mean {v.mean():8.1f}  max {v.max():8.0f}")
        continue
    ok = T[:-1, :, s] > 0
    if not ok.any():
        continue
    v = rel[:, :, s][ok]
    print(f"  {names.get(s, s):28s} mean {v.mean():8.0f}  p50 {np.median(v):8.0f}  p90 {np.percentile(v, 90):8.0f}")
