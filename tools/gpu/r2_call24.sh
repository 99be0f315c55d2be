timeout 600 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -4
rm -f /tmp/t.txt; NTFG_TC_TRACE=/tmp/t.txt timeout 600 python tools/prof_c5.py 1 | tail -1; python tools/tc_wstats.py /tmp/t.txt 2 | grep -v static
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 6 --csv --log-file gpurun_out/r2_l5.csv python tools/prof_c5.py 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 20 --csv --log-file gpurun_out/r2_l2.csv python tools/prof_c2.py 0.5 1 > gpurun_out/r2_l2.log 2>&1
python - <<'PY'
import csv, os, glob
for f in ("gpurun_out/r2_l5.csv","gpurun_out/r2_l2.csv"):
    rows=[r for r in csv.reader(open(f)) if len(r)>10 and r[0].isdigit()]
    print(os.path.basename(f), " ".join("%s:%.3f"%(("K2" if "recon" in r[4] else "K3"), float(r[-1])/1e6) for r in rows))
PY
timeout 900 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-side > gpurun_out/r2_bench9.json 2> gpurun_out/r2_bench9.err; echo "bench rc $?"; tail -3 gpurun_out/r2_bench9.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench9.json").read().strip().splitlines()[-1])
for k in ("value","ms_per_step","clocks","final_loss"): print(k, json.dumps(d.get(k))[:300])
print(d["roofline"]["frac"], d["roofline"]["avg_launch_ms"])
PY
