"""Per-config measurement (BASELINE.json north_star asks for MP
iterations/s and the HBM-roofline fraction of the update and the argmax for every
config).  Dev tool run on the B200; writes profiles/<tag>_configs.{json,md}.

For every config C0..C4 and precision: the loop of one full decomposition (to the
config's stop rule) timed with the library's CUDA events (median of the runs), the
algorithmic update bytes (48 B fp64 / 24 B fp32 per touched
coefficient, counted from the atom list), the per-phase cycle split of CTA 0
(profile mode bit 0) into update and argmax (selection + refresh + exchange), and
the latency floor (profile mode bit 1: the same loop with the update skipped; one-
selection kernel only).

usage: python tools/bench_configs.py [tag] [configs] [precisions] [runs]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import bench
import siggen
from paper_2202_12380_b200.mpgabor import MPGabor

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["C0", "C1", "C2", "C3", "C4"]
precs = sys.argv[3].split(",") if len(sys.argv) > 3 else ["f64", "f32"]
runs = int(sys.argv[4]) if len(sys.argv) > 4 else 3
peak, peak_kind = bench.peaks()
rows = []
for name in cfgs:
    cfg = siggen.CONFIGS[name]
    x = siggen.signal(cfg)
    xd = torch.from_numpy(x).cuda()
    for prec in precs:
        mp = MPGabor(cfg.dicts, cfg.thr, prec)
        W = len(cfg.dicts)
        bench.mp_boxes.clear()
        for u in range(W):
            for v in range(W):
                bench.mp_boxes[(u, v)] = mp.kernel_box(u, v)[0]
        bufs = mp.alloc(cfg.maxit, cfg.Ls)
        batches = [0, None]
        while batches:
            batch = batches.pop(0)
            if batch is None:   # the kernel the automatic choice did not take
                batch = 8 if rows[-1]["kernel"] == "mp_loop_kernel" else 1
            mp.set_batch(batch)
            mp.set_profile(0)
            mp.run(xd, cfg.maxit, cfg.errdb, bufs=bufs, fetch=False)
            loops, dgts = [], []
            for _ in range(runs):
                res, _ = mp.run(xd, cfg.maxit, cfg.errdb, bufs=bufs, fetch=False)
                d, _, lm = mp.last_timing()
                loops.append(lm)
                dgts.append(d)
            out = mp.run(xd, cfg.maxit, cfg.errdb, bufs=bufs)
            n = out.n
            loop_ms = float(np.median(loops))
            kernel = "mp_loop_kernel" if out.rounds == n + 1 else "mp_multi_kernel"
            touched = bench.touched_per_atom(mp, cfg.dicts, out.atoms)
            bpc = 48 if prec == "f64" else 24
            alg = float(touched.sum()) * bpc
            us_it = 1e3 * loop_ms / max(n, 1)
            row = {"config": name, "precision": prec, "batch": batch, "kernel": kernel,
                   "launch": mp.launch_info(), "atoms": int(n), "stop": out.stop_name,
                   "rounds": int(out.rounds), "loop_ms": loop_ms, "dgt_ms": float(np.median(dgts)),
                   "it_per_s": n / (loop_ms * 1e-3), "us_per_it": us_it,
                   "touched_per_it": float(touched.mean()), "alg_bytes_per_it": alg / max(n, 1),
                   "achieved_gbs": alg / (loop_ms * 1e-3) / 1e9}
            row["roofline_frac"] = row["achieved_gbs"] / peak
            # phase split of CTA 0 / thread 0 (profile mode bit 0)
            mp.set_profile(1)
            mp.run(xd, cfg.maxit, cfg.errdb, bufs=bufs, fetch=False)
            c = mp.last_profile()
            mp.set_profile(0)
            if kernel == "mp_loop_kernel":
                upd = c[3] + c[4]
                tot = sum(c[:7])
            else:
                upd = c[11]
                tot = sum(c[:15])
            share = upd / tot if tot else float("nan")
            row["update_share"] = share
            row["update_us_per_it"] = us_it * share
            row["argmax_us_per_it"] = us_it * (1 - share)
            row["update_gbs"] = row["alg_bytes_per_it"] / (row["update_us_per_it"] * 1e-6) / 1e9
            row["update_roofline_frac"] = row["update_gbs"] / peak
            # latency floor (profile mode bit 1): the same loop kernel and launch with the
            # update skipped -- one-selection: the per-iteration exchange/selection chain;
            # multi-selection: rounds of one atom with no items (the fixed cost of a round),
            # scaled by the real run's rounds.  Warm, median of the runs.
            mp.set_profile(2)
            nf = n if kernel == "mp_loop_kernel" else int(out.rounds)
            mp.run(xd, nf, -float("inf"), bufs=bufs, fetch=False)
            fl = []
            for _ in range(runs):
                rf, _ = mp.run(xd, nf, -float("inf"), bufs=bufs, fetch=False)
                fl.append(mp.last_timing()[2] / max(rf.n_atoms, 1))
            mp.set_profile(0)
            per = float(np.median(fl)) * 1e3          # us per floor iteration / round
            row["floor_us_per_round"] = per
            row["floor_us_per_it"] = per * (1.0 if kernel == "mp_loop_kernel" else out.rounds / max(n, 1))
            row["floor_frac"] = row["floor_us_per_it"] / us_it
            rows.append(row)
            print(json.dumps(row), flush=True)
        mp.close()

os.makedirs("profiles", exist_ok=True)
json.dump({"peak_gbs": peak, "peak_kind": peak_kind, "rows": rows}, open(f"profiles/{tag}_configs.json", "w"), indent=1)
with open(f"profiles/{tag}_configs.md", "w") as f:
    f.write(f"# Per-config loop measurements ({tag}, B200, HBM peak {peak:.0f} GB/s {peak_kind})\n\n")
    f.write("batch 0 = automatic kernel choice (the library default), 1 = one selection per iteration, "
            "8 = exact multi-selection.  Loop only (DGT separate); median of the runs.  Update/argmax split "
            "from CTA 0's per-phase clock64 sums.  Roofline = algorithmic update bytes / time / peak.\n\n")
    f.write("| config | prec | batch | kernel | CTAs | TW | atoms | rounds | it/s | us/it | touched/it | GB/s | frac | "
            "update us/it | update frac | argmax us/it | floor us/it | floor frac | DGT ms |\n")
    f.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        fl = r.get("floor_us_per_it")
        f.write(f"| {r['config']} | {r['precision']} | {r['batch']} | {r['kernel']} | {r['launch']['cluster']} | {r['launch']['tile_width']} | {r['atoms']} | {r['rounds']} | "
                f"{r['it_per_s']:.0f} | {r['us_per_it']:.3f} | {r['touched_per_it']:.0f} | {r['achieved_gbs']:.1f} | "
                f"{r['roofline_frac']:.4f} | {r['update_us_per_it']:.3f} | {r['update_roofline_frac']:.4f} | "
                f"{r['argmax_us_per_it']:.3f} | {'' if fl is None else f'{fl:.3f}'} | "
                f"{r.get('floor_frac', float('nan')):.2f} | {r['dgt_ms']:.2f} |\n")
print("wrote", f"profiles/{tag}_configs.md")
