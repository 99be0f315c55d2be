timeout 3000 python -m pytest tests -m gpu -x -q --durations=8 -p no:cacheprovider > gpurun_out/r2_gputests2.log 2>&1; echo "tests rc $?"; tail -15 gpurun_out/r2_gputests2.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench5.json 2> gpurun_out/r2_bench5.err; echo "bench rc $?"; tail -3 gpurun_out/r2_bench5.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench5.json").read().strip().splitlines()[-1])
for k,v in d.items(): print(k, json.dumps(v)[:900])
PY
