timeout 600 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 300 python tools/precision_probe.py c2q 2>&1 | grep -v Warn
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo "bench rc $?"; tail -3 gpurun_out/r2_bench2.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench2.json").read().strip().splitlines()[-1])
for k in ("value","ms_per_step","roofline","whole_step"): print(k, json.dumps(d.get(k))[:700])
for k in ("c2",): print(k, json.dumps(d.get(k))[:1500])
PY
g++ -std=c++20 -O1 -g -fsanitize=address -fno-omit-frame-pointer -Iinclude tests/cpp/dropin_test.cpp paper_2602_14683_b200/csrc/ntf_api.cpp -Lpaper_2602_14683_b200/lib_asan -lntfg -Wl,-rpath,$PWD/paper_2602_14683_b200/lib_asan -o /tmp/dropin_asan && ASAN_OPTIONS=protect_shadow_gap=0:detect_leaks=0 timeout 300 /tmp/dropin_asan 2>&1 | grep -v "^stage" | head -60
