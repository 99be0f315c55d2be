timeout 600 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
for cfgv in "0 0" "5 2" "4 2" "3 4"; do
  set -- $cfgv
  NTFG_TC_NST=$1 NTFG_TC_GD=$2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 6 --csv --log-file gpurun_out/r2_l5_$1_$2.csv python tools/prof_c5.py 1 > /dev/null 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 20 --csv --log-file gpurun_out/r2_l2.csv python tools/prof_c2.py 0.5 1 > gpurun_out/r2_l2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 20 --csv --log-file gpurun_out/r2_l2b1.csv python tools/prof_c2.py 1.0 1 > /dev/null 2>&1
python - <<'PY'
import csv, os, glob
for f in sorted(glob.glob("gpurun_out/r2_l*.csv")):
    rows=[r for r in csv.reader(open(f)) if len(r)>10 and r[0].isdigit()]
    print(os.path.basename(f), " ".join("%s:%.3f"%(("K2" if "recon" in r[4] else "K3"), float(r[-1])/1e6) for r in rows))
PY
