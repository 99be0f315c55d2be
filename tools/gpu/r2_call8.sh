timeout 600 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
rm -f /tmp/t.txt; NTFG_TC_TRACE=/tmp/t.txt timeout 600 python tools/prof_c5.py 1 | tail -1; python tools/tc_wstats.py /tmp/t.txt 4
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench4.json 2> gpurun_out/r2_bench4.err; echo "bench rc $?"; tail -3 gpurun_out/r2_bench4.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench4.json").read().strip().splitlines()[-1])
for k in ("value","ms_per_step","roofline","whole_step"): print(k, json.dumps(d.get(k))[:700])
for k in ("c2",): print(k, json.dumps(d.get(k))[:1500])
PY
