timeout 3000 python -m pytest tests -m gpu -x -q --durations=6 -p no:cacheprovider > gpurun_out/r2_gputests3.log 2>&1; echo "tests rc $?"; tail -12 gpurun_out/r2_gputests3.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python bench.py --steps 20 --warmup 3 > gpurun_out/r2_bench8.json 2> gpurun_out/r2_bench8.err; echo "bench rc $?"; tail -3 gpurun_out/r2_bench8.err
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench8.json").read().strip().splitlines()[-1])
for k,v in d.items(): print(k, json.dumps(v)[:700])
PY
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench8_ref.json 2>/dev/null; cut -c1-400 gpurun_out/r2_bench8_ref.json
