rm -f /tmp/t.txt; NTFG_TC_TRACE=/tmp/t.txt timeout 600 python tools/prof_c5.py 1 | tail -1; python tools/tc_wstats.py /tmp/t.txt 4
for cfgv in "3 2" "4 2" "5 2"; do set -- $cfgv
NTFG_TC_NST=$1 NTFG_TC_GD=$2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract" -c 4 --csv --log-file gpurun_out/r2_l5_$1.csv python tools/prof_c5.py 1 > /dev/null 2>&1
done
NTFG_TC_SEG=8 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract" -c 4 --csv --log-file gpurun_out/r2_l5_seg8.csv python tools/prof_c5.py 1 > /dev/null 2>&1
python - <<'PY'
import csv, os, glob
for f in sorted(glob.glob("gpurun_out/r2_l5_[345s]*.csv")):
    rows=[r for r in csv.reader(open(f)) if len(r)>10 and r[0].isdigit()]
    print(os.path.basename(f), " ".join("%.3f"%(float(r[-1])/1e6) for r in rows))
PY
