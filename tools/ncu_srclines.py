"""Dev tool: per-source-line warp-stall samples from an `ncu --page source --csv --print-source
cuda,sass` export (file:line, samples, top stall reasons).  usage: ncu_srclines.py export.csv [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname, hdr, agg = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[2:], r[2:]))
    try:
        s = int(d.get("Warp Stall Sampling (All Samples)", "0"))
    except ValueError:
        continue
    stalls = {k: int(v) for k, v in d.items() if k.startswith("stall_") and "Not Issued" not in k and v.isdigit()}
    agg.append((s, fname, int(r[0]), r[1][:70], stalls))
tot = sum(a[0] for a in agg)
agg.sort(key=lambda a: -a[0])
print(f"total samples {tot}")
for s, f, ln, src, st in agg[:top]:
    tops = ", ".join(f"{k[6:]} {v}" for k, v in sorted(st.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<5d} {src:70s} | {tops}")
