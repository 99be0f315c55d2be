timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py tests/test_tucker_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 6 --csv --log-file gpurun_out/r2_l5.csv python tools/prof_c5.py 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"tc_contract|recon_t" -c 20 --csv --log-file gpurun_out/r2_l2.csv python tools/prof_c2.py 0.5 1 > gpurun_out/r2_l2.log 2>&1
python - <<'PY'
import csv, os
for f in ("gpurun_out/r2_l5.csv","gpurun_out/r2_l2.csv"):
    rows=[r for r in csv.reader(open(f)) if len(r)>10 and r[0].isdigit()]
    print(os.path.basename(f), " ".join("%s:%.3f"%(("K2" if "recon" in r[4] else "K3"), float(r[-1])/1e6) for r in rows))
PY
timeout 1500 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench11.json 2> gpurun_out/r2_bench11.err; echo "bench rc $?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/r2_bench11.json").read().strip().splitlines()[-1])
print("value", d["value"], d["ms_per_step"], d["clocks"])
print("roofline", d["roofline"]["frac"], d["roofline"]["avg_launch_ms"], d["whole_step"]["kernel_ms_one_eager_outer"])
print("c2", {k:round(v["outer_it_per_s"],1) for k,v in d["c2"]["per_beta"].items()}, d["c2"]["roofline_k3"]["frac"], d["c2"]["kernel_ms_per_outer"])
print("c3", {k:round(v["it_per_s"],1) for k,v in d["c3"]["fits"].items()})
PY
