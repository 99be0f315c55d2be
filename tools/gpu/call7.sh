python tools/tc_ablate.py 0.5 2>&1 | grep -v Warn | head -4
for sk in 0 3; do
  out=gpurun_out/c5k3_skip$sk
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_contract_kernel --launch-skip $sk -c 1 -o $out python tools/prof_c5.py 1 > $out.ncu.log 2>&1
  python tools/ncu_summary.py $out.ncu-rep > $out.summary.txt 2>&1
  ncu -i $out.ncu-rep --page source --csv --print-source cuda > $out.src.csv 2>/dev/null
  python tools/ncu_lines.py $out.src.csv 45 > $out.lines.txt 2>&1
  ncu -i $out.ncu-rep --page raw --csv > $out.raw.csv 2>/dev/null
  gzip -f $out.src.csv; rm -f $out.ncu-rep
  cat $out.summary.txt; head -50 $out.lines.txt
done
