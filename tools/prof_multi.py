"""Dev tool: per-phase time per round of the multi-selection loop (profile mode bit 0).

Slots (mpgabor.h, mpgabor_last_profile): 0 wait, 1 verify, 2 bar, 3 rank, 4 bar, 5 geometry,
6 bar, 7 pairwise, 8 bar, 9 walk, 10 bar, 11 own items, 12 bar+lvl1+bar, 13 top-K, 14 push; 15 rounds.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

PH = ["wait", "verify", "b", "rank", "geom+b", "pair", "b", "-", "-", "scan", "b", "items", "lvl1", "topk", "push"]
cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C2"]
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100000
batches = [int(b) for b in sys.argv[3].split(",")] if len(sys.argv) > 3 else [8]
prec = sys.argv[4] if len(sys.argv) > 4 else "f64"
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    xd = torch.from_numpy(siggen.signal(cfg)).cuda()
    mp = MPGabor(cfg.dicts, cfg.thr, prec)
    for b in batches:
        mp.set_batch(b)
        mp.set_profile(1)
        mp.run(xd, K, cfg.errdb, fetch=False)
        res, _ = mp.run(xd, K, cfg.errdb, fetch=False)
        c = mp.last_profile()
        loop = mp.last_timing()[2]
        n = max(1, c[15] if b != 1 else c[7])
        print(f"{name} {prec} batch={b}: atoms {res.n_atoms} rounds {n} loop {loop:.2f} ms "
              f"({1e3 * loop / n:.3f} us/round, {1e3 * loop / max(res.n_atoms, 1):.3f} us/atom) | "
              + " ".join(f"{p}={x / n:.0f}" for p, x in zip(PH, c[:15])) + " cycles/round", flush=True)
        print(f"   walk: mean last window position {c[20] / n:.1f}; ends: B {c[21]} window {c[22]} "
              f"list-exhausted {c[23]} zero/stop {c[24]} overlap {c[25]} last-entry {c[26]}", flush=True)
        print(f"   warp 1: wait {c[30] / n:.0f} rank {c[31] / n:.0f}", flush=True)
        print(f"   walk split: setup {c[29] / n:.0f} bitmask {c[27] / n:.0f} E+atoms {c[28] / n:.0f} item-scan {c[9] / n:.0f}", flush=True)
        print("   top-K per level (pops / barrier / merge / barrier): " + " | ".join(
            " ".join(f"{c[32 + 4 * L + i] / n:.0f}" for i in range(4)) for L in range(3)), flush=True)
        print(f"   roll-back rounds {c[56]} ({100 * c[56] / n:.1f} % of rounds); first rejected candidate 1..7: "
              + " ".join(str(c[56 + i]) for i in range(1, 8)), flush=True)
        Cn = min(128, mp.launch_info()["cluster"])
        busy = [c[64 + r] / n for r in range(Cn)]
        items = [c[192 + r] / n for r in range(Cn)]
        print(f"   per-CTA busy cycles/round (receive -> publish) over {Cn} CTAs: mean {sum(busy) / Cn:.0f} "
              f"min {min(busy):.0f} max {max(busy):.0f}; items/round mean {sum(items) / Cn:.2f} "
              f"min {min(items):.2f} max {max(items):.2f}", flush=True)
        print(f"   candidate-list rebuilds: {c[19]} ({100 * c[19] / n:.2f} % of rounds), "
              f"{c[17] / max(c[19], 1):.0f} cycles each; extraction {c[16] / n:.0f} cycles/round", flush=True)
        rb = [c[320 + r] for r in range(Cn)]
        print(f"   rebuilds over {Cn} CTAs: total {sum(rb)} ({100 * sum(rb) / n:.1f} % of rounds if disjoint), "
              f"min {min(rb)} max {max(rb)}", flush=True)
        labels = ["<1k", "1-2k", "2-3k", "3-4k", "4-6k", "6-8k", "8-12k", ">=12k"]
        print("   CTA 0 message waits: " + " ".join(
            f"{labels[i]}: {c[448 + i]} ({c[456 + i] / max(c[448 + i], 1):.0f})" for i in range(8))
              + f"; share of wait cycles in rounds waiting >= 4k: "
              f"{sum(c[460:464]) / max(sum(c[456:464]), 1):.2f}", flush=True)
        nc = max(c[472], 1)
        print(f"   rebuild split (CTA 0, cycles per rebuild): node maxima {c[468] / nc:.0f}, rank counts {c[469] / nc:.0f}, "
              f"gathers {c[470] / nc:.0f}, retries {c[471] / nc:.2f} per rebuild; record scans (list short) {c[473]}", flush=True)
        print("   CTA-rounds by items (buckets of 8): " + " ".join(str(c[480 + i]) for i in range(16)), flush=True)
        print("   CTA-rounds by busy cycles (buckets of 4096): " + " ".join(str(c[496 + i]) for i in range(16)), flush=True)
        print("   deepest CTA-list position in the walk window (0..3): "
              + " ".join(str(c[464 + i]) for i in range(4)), flush=True)
        mp.set_profile(0)
    mp.close()
