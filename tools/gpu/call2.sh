python tools/precision_probe.py c2 2>&1 | grep -v Warn
NTFG_DISABLE_TC=1 python tools/precision_probe.py c2 2>&1 | grep -v Warn | sed 's/^/NOTC /' | head -8
python tools/precision_probe.py c5 2>&1 | grep -v Warn
