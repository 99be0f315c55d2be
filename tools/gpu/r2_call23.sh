rm -f /tmp/t.txt; NTFG_TC_TRACE=/tmp/t.txt timeout 600 python tools/prof_c5.py 1 | tail -1; python tools/tc_wstats.py /tmp/t.txt 4
