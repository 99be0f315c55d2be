#!/bin/bash
# Box-side ncu --set full capture of ONE kernel (regex $2) of command "${@:3}",
# reduced to small text summaries (the .ncu-rep of a 15k-instruction kernel
# with source is ~50 MB; kept only when $KEEP_REP=1).
# usage: tools/ncu_capture.sh NAME REGEX cmd...
set -e
name=$1; rx=$2; shift 2
out=gpurun_out/$name
ncu --set full --clock-control none --import-source on -k "regex:$rx" -c 1 -o "$out" "$@" > "$out.ncu.log" 2>&1
python tools/ncu_summary.py "$out.ncu-rep" > "$out.summary.txt" 2>&1 || true
ncu -i "$out.ncu-rep" --page source --csv --print-source sass > "$out.sass.csv" 2>/dev/null || true
python tools/sass_hist.py "$out.sass.csv" 30 > "$out.sass_hist.txt" 2>&1 || true
ncu -i "$out.ncu-rep" --page raw --csv > "$out.raw.csv" 2>/dev/null || true
gzip -f "$out.sass.csv"
[ "${KEEP_REP:-0}" = "1" ] || rm -f "$out.ncu-rep"
