"""Summarise NTFG_TC_TRACE output (clock64 events of tc_contract_kernel):
per launch, median per-unit MMA time, epilogue time, and MMA waits.
usage: NTFG_TC_TRACE=/tmp/t.txt python tools/prof_c2.py 0.5 1; python tools/tc_trace.py /tmp/t.txt"""
import statistics as S
import sys

launches, cur = [], None
for line in open(sys.argv[1]):
    if line.startswith("launch"):
        cur = [line.strip(), [], []]
        launches.append(cur)
    elif line.startswith("wstats"):
        cur[2].append([int(x) for x in line.split()[1:]])
    else:
        v = [int(x) for x in line.split()]
        if v[5]:  # MMA side recorded
            cur[1].append(v)
for hdr, rows, ws in launches[:6]:
    if not rows:
        continue
    mma = [r[9] - r[5] for r in rows]           # unit MMA span (after acc_empty -> last commit)
    wait_empty = [r[5] - r[4] for r in rows]     # MMA waiting for the accumulator buffer
    epi = [r[3] - r[2] for r in rows if r[3]]    # epilogue span
    epi_lag = [r[2] - r[9] for r in rows if r[2]]  # commit -> epilogue start
    wa = [r[6] for r in rows]
    wb = [r[7] for r in rows]
    med = lambda x: int(S.median(x)) if x else -1
    print(hdr)
    print("  unit MMA span %d  wait acc_empty %d  wait a_full %d  wait b_full %d  epilogue %d  commit->epi %d"
          % (med(mma), med(wait_empty), med(wa), med(wb), med(epi), med(epi_lag)))
    if ws:
        m = [med([w[i] for w in ws]) for i in range(7)]
        print("  B: wait g_full %d wait empty %d total %d | gather: wait g_empty %d total %d | TMA: wait empty %d total %d"
              % tuple(m))
