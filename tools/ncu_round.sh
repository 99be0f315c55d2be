#!/bin/bash
# Round evidence (box side): launch lists (ncu --metrics gpu__time_duration.sum) of one eager outer
# iteration per config, and one ncu --set full capture of each hot kernel, reduced to text summaries
# under gpurun_out/prof_$TAG/.  Copy what should be judged into profiles/.
# usage: tools/ncu_round.sh TAG
TAG=${1:-r02}
out=gpurun_out/prof_$TAG
mkdir -p $out
list() {  # name cmd...
  name=$1; shift
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $out/$name.launches.csv "$@" > $out/$name.launches.log 2>&1
  python - $out/$name.launches.csv > $out/$name.launches.txt <<'PY'
import csv, sys, collections
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>10 and r[0].isdigit()]
agg=collections.defaultdict(lambda:[0,0.0])
for r in rows:
    name=r[4].split("(")[0][:70]
    agg[name][0]+=1; agg[name][1]+=float(r[-1])/1e3
tot=sum(v[1] for v in agg.values())
print("launches", len(rows), "total_us %.1f (ncu per-launch times are cold-cache and serialised)"%tot)
for k,v in sorted(agg.items(), key=lambda kv:-kv[1][1]): print("%-70s n=%4d %10.1f us %5.1f%% avg %.1f us"%(k,v[0],v[1],100*v[1]/tot,v[1]/v[0]))
PY
}
full() {  # name regex skip cmd...
  name=$1; rx=$2; skip=$3; shift 3
  timeout 1500 ncu --set full --clock-control none --import-source on -k regex:$rx --launch-skip $skip -c 1 -o $out/$name "$@" > $out/$name.ncu.log 2>&1
  python tools/ncu_summary.py $out/$name.ncu-rep > $out/$name.summary.txt 2>&1
  ncu -i $out/$name.ncu-rep --page source --csv --print-source sass > $out/$name.sass.csv 2>/dev/null
  python tools/sass_hist.py $out/$name.sass.csv 24 > $out/$name.sass_hist.txt 2>&1
  ncu -i $out/$name.ncu-rep --page raw --csv > $out/$name.raw.csv 2>/dev/null
  rm -f $out/$name.sass.csv $out/$name.ncu-rep
}
list bench python bench.py --steps 2 --warmup 3 --no-side --no-e2e --no-cpu-baseline
list c5 python tools/prof_c5.py 1
list c2_b05 python tools/prof_c2.py 0.5 1
list c2_b1 python tools/prof_c2.py 1.0 1
list c3_jcomm python tools/prof_c3.py jcomm 0.5 1
list c3_bcomm python tools/prof_c3.py bcomm 0.5 1
list c4 python tools/prof_c4.py 2
full c5_k3 tc_contract_kernel 1 python tools/prof_c5.py 1
full c5_k2 recon_tc_kernel 0 python tools/prof_c5.py 1
full c2_k3 tc_contract_kernel 1 python tools/prof_c2.py 0.5 1
full c2_k2 recon_tc_kernel 0 python tools/prof_c2.py 0.5 1
full c3_rowgemm rowgemm_tiled_kernel 1 python tools/prof_c3.py jcomm 0.5 1
full c3_recon recon_tc_kernel 0 python tools/prof_c3.py jcomm 0.5 1
full c4_coo coo_piece 4 python tools/prof_c4.py 2
python - $out <<'PY'
import csv, json, sys, os, glob
out=sys.argv[1]; res={}
for f in sorted(glob.glob(out+"/*.raw.csv")):
    rows=list(csv.reader(open(f)))
    if len(rows)<3: continue
    h=rows[0]; r=rows[2]
    g=lambda m: float(r[h.index(m)].replace(",","")) if m in h and r[h.index(m)] else None
    unit=lambda m: rows[1][h.index(m)] if m in h else ""
    def tobytes(m):
        v=g(m); u=unit(m)
        if v is None: return None
        return v*{"byte":1,"Kbyte":1e3,"Mbyte":1e6,"Gbyte":1e9,"Tbyte":1e12}.get(u,1)
    key=os.path.basename(f)[:-8]
    rd,wr=tobytes("dram__bytes_read.sum"),tobytes("dram__bytes_write.sum")
    res[key]={"kernel":r[h.index("Kernel Name")][:80],"dram_bytes_per_launch":(rd or 0)+(wr or 0),"dram_read":rd,"dram_write":wr,
              "duration_us":(g("gpu__time_duration.sum") or 0)*{"nsecond":1e-3,"usecond":1.0,"msecond":1e3,"second":1e6}.get(unit("gpu__time_duration.sum"),1.0),"l2_bytes":tobytes("lts__t_bytes.sum"),"source":"ncu --set full, tools/ncu_round.sh"}
json.dump(res, open(out+"/ncu_traffic.json","w"), indent=1)
print(json.dumps(res, indent=1))
PY
[ -x tools/mma_probe ] || nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_probe tools/mma_probe.cu -lcuda
./tools/mma_probe > $out/mma_probe.txt 2>&1
for f in $out/*.summary.txt $out/*.launches.txt; do echo "=== $f"; head -30 $f; done
