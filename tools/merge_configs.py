"""Dev tool: merge per-config rows (tools/bench_configs.py output) into profiles/<tag>_configs.*:
rows of the same (config, precision) are replaced.  usage: python tools/merge_configs.py <tag> <new.json>..."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
tag = sys.argv[1]
base = json.load(open(f"profiles/{tag}_configs.json"))
rows = base["rows"]
for fn in sys.argv[2:]:
    new = json.load(open(fn))["rows"]
    keys = {(r["config"], r["precision"]) for r in new}
    rows = [r for r in rows if (r["config"], r["precision"]) not in keys] + new
order = {c: i for i, c in enumerate(["C0", "C1", "C2", "C3", "C4"])}
rows.sort(key=lambda r: (order.get(r["config"], 9), r["precision"] != "f64", r["batch"] != 0))
base["rows"] = rows
json.dump(base, open(f"profiles/{tag}_configs.json", "w"), indent=1)
peak, kind = base["peak_gbs"], base["peak_kind"]
with open(f"profiles/{tag}_configs.md", "w") as f:
    f.write(f"# Per-config loop measurements ({tag}, B200, HBM peak {peak:.0f} GB/s {kind})\n\n")
    f.write("batch 0 = automatic kernel choice (the library default), 1 = one selection per iteration, "
            "8 = exact multi-selection.  Loop only (DGT separate); median of the runs.  Update/argmax split "
            "from CTA 0's per-phase clock64 sums.  Roofline = algorithmic update bytes / time / peak.\n\n")
    f.write("| config | prec | batch | kernel | CTAs | TW | atoms | rounds | it/s | us/it | touched/it | GB/s | frac | "
            "update us/it | update frac | argmax us/it | floor us/it | DGT ms |\n")
    f.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        fl = r.get("floor_us_per_it")
        f.write(f"| {r['config']} | {r['precision']} | {r['batch']} | {r['kernel']} | {r['launch']['cluster']} | "
                f"{r['launch']['tile_width']} | {r['atoms']} | {r['rounds']} | "
                f"{r['it_per_s']:.0f} | {r['us_per_it']:.3f} | {r['touched_per_it']:.0f} | {r['achieved_gbs']:.1f} | "
                f"{r['roofline_frac']:.4f} | {r['update_us_per_it']:.3f} | {r['update_roofline_frac']:.4f} | "
                f"{r['argmax_us_per_it']:.3f} | {'' if fl is None else f'{fl:.3f}'} | {r['dgt_ms']:.2f} |\n")
print("merged", len(rows), "rows")
