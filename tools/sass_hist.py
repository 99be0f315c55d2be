"""Opcode histogram (instructions executed, stall samples) of one kernel's
SASS source page: ncu -i REP --page source --csv --print-source sass > CSV.
usage: python tools/sass_hist.py CSV [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
i = 0
while i < len(rows):
    if rows[i] and rows[i][0] == "Kernel Name":
        name = rows[i][1]
        hdr = rows[i + 1]
        ie = hdr.index("Instructions Executed")
        sm = hdr.index("Warp Stall Sampling (All Samples)")
        op, st, tot, j = collections.Counter(), collections.Counter(), 0, i + 2
        while j < len(rows) and rows[j] and rows[j][0] != "Kernel Name":
            r = rows[j]
            if len(r) > ie and r[1].strip():
                toks = r[1].strip().split()
                o = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
                o = o.split(".")[0]
                n = int(r[ie] or 0)
                op[o] += n
                st[o] += int(r[sm] or 0)
                tot += n
            j += 1
        print(name[:110], "warp-instructions", tot)
        for o, n in op.most_common(top):
            print(f"  {o:10s} {n:12d} {100.0 * n / max(tot, 1):5.1f}%  stall-samples {st[o]}")
        i = j
    else:
        i += 1
