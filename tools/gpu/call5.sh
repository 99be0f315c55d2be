timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py tests/test_tucker_gpu.py tests/test_extrap_api.py tests/test_dropin_cpp.py tests/test_dist_gpu.py -q -x 2>&1 | tail -15
timeout 300 python tools/precision_probe.py c2q 2>&1 | grep -v Warn
timeout 300 python tools/precision_probe.py c5q 2>&1 | grep -v Warn
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err; echo "bench rc $?"; tail -5 gpurun_out/bench5.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench5.json").read().strip().splitlines()[-1])
for k in ("value","ms_per_step","roofline","whole_step","cpu_baseline","e2e","clocks","gpu_launches"): print(k, json.dumps(d.get(k))[:700])
for k in ("c2","c1","c3","c4_sparse"): print(k, json.dumps(d.get(k))[:1200])
PY
