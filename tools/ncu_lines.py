"""Top source lines by warp-stall samples from an ncu source page
(ncu -i REP --page source --csv --print-source cuda ...).
usage: python tools/ncu_lines.py CSV [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr_i = next(i for i, r in enumerate(rows) if r and any("Warp Stall Sampling (All Samples)" == c for c in r))
hdr = rows[hdr_i]
si = hdr.index("Warp Stall Sampling (All Samples)")
src_i = hdr.index("Source") if "Source" in hdr else 1
li = hdr.index("#") if "#" in hdr else 0
ie = hdr.index("Instructions Executed") if "Instructions Executed" in hdr else None
data = []
tot = 0
for r in rows[hdr_i + 1:]:
    if len(r) <= si:
        continue
    try:
        v = int(float(r[si] or 0))
    except ValueError:
        continue
    tot += v
    data.append((v, r[li], r[src_i].strip()[:110], r[ie] if ie is not None else ""))
print("total stall samples", tot)
for v, ln, src, n in sorted(data, reverse=True)[:top]:
    print(f"{100.0 * v / max(tot, 1):5.1f}%  L{ln:>5}  inst {n:>10}  {src}")
