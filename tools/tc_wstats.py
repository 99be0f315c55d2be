"""Per-launch medians of the role wait counters of tc_contract_kernel (NTFG_TC_TRACE file):
B producers (wait gathers / wait slot / total), gather warp (wait / total), TMA producer (wait / total), in cycles.
The counters are compiled in only by a trace build:
  NTFG_TC_TRACE_BUILD=1 python -c "from paper_2602_14683_b200 import build as B; B.build(force=True)"
usage: NTFG_TC_TRACE=/tmp/t.txt python tools/prof_c5.py 1; python tools/tc_wstats.py /tmp/t.txt"""
import statistics as S
import sys

launches, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("launch"):
        cur = [line.strip(), []]
        launches.append(cur)
    elif line.startswith("wstats"):
        cur[1].append([int(x) for x in line.split()[1:]])
for hdr, ws in launches[: int(sys.argv[2]) if len(sys.argv) > 2 else 6]:
    if not ws:
        continue
    m = [int(S.median([w[i] for w in ws])) for i in range(7)]
    print(hdr)
    print("  B: wait g_full %d  wait empty %d  total %d | gather: wait g_empty %d  total %d | TMA: wait empty %d  total %d" % tuple(m))
    print("  (static-B launches: the three B slots are the epilogue's wait for finished tiles, its drain cycles, and the issuer's wait for drains)")
