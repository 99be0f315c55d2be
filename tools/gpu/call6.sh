python tools/tc_ablate.py 0.5 2>&1 | grep -v Warn
WORKLOAD=c5 python tools/tc_ablate.py 0.5 2>&1 | grep -v Warn
