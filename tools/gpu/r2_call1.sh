set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 3000 python -m pytest tests -m gpu -x -q --durations=15 -p no:cacheprovider > gpurun_out/r2_gputests.log 2>&1; echo "tests rc $?"; tail -30 gpurun_out/r2_gputests.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo "bench rc $?"; tail -5 gpurun_out/r2_bench1.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench1.json").read().strip().splitlines()[-1])
for k,v in d.items(): print(k, json.dumps(v)[:1200])
PY
