timeout 900 python -m pytest tests/test_tucker_gpu.py tests/test_unfold_gpu.py tests/test_tc_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -4
timeout 900 python -m pytest tests/test_config_parity_gpu.py -x -q -k "c3" -p no:cacheprovider 2>&1 | tail -3
for a in jcomm bcomm; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_c3_$a.csv python tools/prof_c3.py $a 0.5 1 > gpurun_out/r2_c3_$a.log 2>&1
python - $a <<'PY'
import csv, sys, collections
a=sys.argv[1]
rows=[r for r in csv.reader(open("gpurun_out/r2_c3_%s.csv"%a)) if len(r)>10 and r[0].isdigit()]
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    name=r[4].split("(")[0][:60]
    agg[name][0]+=1; agg[name][1]+=float(r[-1])/1e3
tot=sum(v[1] for v in agg.values())
print(a, "launches", len(rows), "total us %.1f"%tot)
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1])[:10]: print("  %-60s n=%3d  %9.1f us  %5.1f%%"%(k,v[0],v[1],100*v[1]/tot))
PY
done
