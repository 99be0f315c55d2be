timeout 600 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
rm -f /tmp/t.txt; NTFG_TC_TRACE=/tmp/t.txt timeout 600 python tools/prof_c5.py 1 | tail -1; python tools/tc_wstats.py /tmp/t.txt 4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 12 --csv --log-file gpurun_out/r2_l5.csv python tools/prof_c5.py 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 20 --csv --log-file gpurun_out/r2_l2.csv python tools/prof_c2.py 0.5 1 > gpurun_out/r2_l2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 20 --csv --log-file gpurun_out/r2_l2b1.csv python tools/prof_c2.py 1.0 1 > /dev/null 2>&1
python - <<'PY'
import csv, os
for f in ("r2_l5","r2_l2","r2_l2b1"):
    if not os.path.exists("gpurun_out/%s.csv"%f): print(f, "missing"); continue
    rows=[r for r in csv.reader(open("gpurun_out/%s.csv"%f)) if len(r)>10 and r[0].isdigit()]
    print(f, " ".join("%s:%.3f"%(("K2" if "recon" in r[4] else "K3"), float(r[-1])/1e6) for r in rows))
PY
tail -3 gpurun_out/r2_l2.log
