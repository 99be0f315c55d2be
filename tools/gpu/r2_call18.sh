timeout 900 python -m pytest tests/test_tucker_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 1500 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench7.json 2> gpurun_out/r2_bench7.err; echo "bench rc $?"; tail -3 gpurun_out/r2_bench7.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench7.json").read().strip().splitlines()[-1])
for k,v in d.items(): print(k, json.dumps(v)[:1500])
PY
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2_bench7_ref.json 2>/dev/null; cat gpurun_out/r2_bench7_ref.json | cut -c1-600
