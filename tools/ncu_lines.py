"""Dev tool: aggregate an ncu SASS source page per CUDA source line.

usage: python tools/ncu_lines.py <report.ncu-rep> <cubin> <mangled kernel name> [top]
(the cubin comes from `cuobjdump -xelf all libmpgabor.so`; compile with -lineinfo)
"""
import csv
import io
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, ln in enumerate(dis) if ln.startswith(fn + ":"))
end = next((i for i in range(start + 1, len(dis)) if dis[i].startswith("//----") and ".text." in dis[i]), len(dis))
off2line, cur = {}, None
for ln in dis[start:end]:
    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
    if m:
        cur = f"{m.group(1).split('/')[-1]}:{m.group(2)}"
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
    if m and cur:
        off2line[int(m.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
iA, iIE, iST = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
iNI = h.index("Warp Stall Sampling (Not-issued Samples)")
base = int(rows[2][iA], 16)
agg = defaultdict(lambda: [0.0, 0.0, 0.0])
for r in rows[2:]:
    try:
        off = int(r[iA], 16) - base
        a = agg[off2line.get(off, "?")]
        a[0] += float(r[iIE] or 0)
        a[1] += float(r[iST] or 0)
        a[2] += float(r[iNI] or 0)
    except (ValueError, IndexError):
        pass
T = sum(a[0] for a in agg.values())
S = sum(a[1] for a in agg.values())
print(f"instructions {T:.0f}, stall samples {S:.0f}")
for k, a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k:24s} inst {a[0] / T * 100:5.1f}%  samples {a[1] / S * 100:5.1f}%")
