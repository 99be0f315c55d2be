timeout 900 python -m pytest tests/test_tc_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"recon_t" -c 2 --csv --log-file gpurun_out/r2_l5.csv python tools/prof_c5.py 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"recon_t" -c 2 --csv --log-file gpurun_out/r2_l2.csv python tools/prof_c2.py 0.5 1 > gpurun_out/r2_l2.log 2>&1
python - <<'PY'
import csv, os
for f in ("gpurun_out/r2_l5.csv","gpurun_out/r2_l2.csv"):
    rows=[r for r in csv.reader(open(f)) if len(r)>10 and r[0].isdigit()]
    print(os.path.basename(f), " ".join("%s:%.3f"%(("K2" if "recon" in r[4] else "K3"), float(r[-1])/1e6) for r in rows))
PY
