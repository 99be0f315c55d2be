timeout 900 python -m pytest tests/test_coo_gpu.py tests/test_dist_gpu.py tests/test_io_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_c4.csv python tools/prof_c4.py 2 > gpurun_out/r2_c4.log 2>&1
python - <<'PY'
import csv, collections
rows=[r for r in csv.reader(open("gpurun_out/r2_c4.csv")) if len(r)>10 and r[0].isdigit()]
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    name=r[4].split("(")[0][:60]; agg[name][0]+=1; agg[name][1]+=float(r[-1])/1e3
tot=sum(v[1] for v in agg.values())
print("launches", len(rows), "total us %.1f"%tot)
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])[:8]: print("  %-60s n=%3d  %9.1f us  avg %.1f"%(k,v[0],v[1],v[1]/v[0]))
PY
python - <<'PY'
import sys, json
sys.path.insert(0,'.')
import bench, argparse
a=argparse.Namespace(steps=10, warmup=3, no_cpu_baseline=True)
d=bench.Dist(); d.init()
r=bench.run_c4(a,d)
print({k:r[k] for k in ("outer_it_per_s","ms_per_step","final_loss")}, r["e2e"]["value"])
PY
