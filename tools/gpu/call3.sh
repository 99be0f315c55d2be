for u in 16 64 256 1024; do NTFG_TC_UNIT_ROWS=$u python tools/precision_probe.py c2q 2>&1 | grep -v Warn | sed "s/^/U$u /"; done
for u in 256 2048; do NTFG_TC_UNIT_ROWS=$u python tools/precision_probe.py c5q 2>&1 | grep -v Warn | sed "s/^/U$u /"; done
