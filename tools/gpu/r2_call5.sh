timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py tests/test_dropin_cpp.py -x -q -p no:cacheprovider 2>&1 | tail -15
timeout 300 python tools/precision_probe.py c2q 2>&1 | grep -v Warn
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; echo "bench rc $?"; tail -3 gpurun_out/r2_bench3.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench3.json").read().strip().splitlines()[-1])
for k in ("value","ms_per_step","roofline","whole_step"): print(k, json.dumps(d.get(k))[:700])
for k in ("c2",): print(k, json.dumps(d.get(k))[:1500])
PY
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 30 --csv --log-file gpurun_out/r2_c5_launches.csv python tools/prof_c5.py 1 > gpurun_out/r2_c5_ncu.log 2>&1; tail -2 gpurun_out/r2_c5_ncu.log
python - <<'PY'
import csv
rows=[r for r in csv.reader(open("gpurun_out/r2_c5_launches.csv")) if len(r)>10 and r[0].isdigit()]
for r in rows: print(r[4][:40], r[-1])
PY
