for spec in "c5k2:recon_tc_kernel:0" "c5k3:tc_contract_kernel:1"; do
  IFS=: read name rx skip <<< "$spec"
  out=gpurun_out/r2_$name
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:$rx --launch-skip $skip -c 1 -o $out python tools/prof_c5.py 1 > $out.ncu.log 2>&1
  python tools/ncu_summary.py $out.ncu-rep > $out.summary.txt 2>&1
  ncu -i $out.ncu-rep --page source --csv --print-source cuda > $out.src.csv 2>/dev/null
  python tools/ncu_lines.py $out.src.csv 45 > $out.lines.txt 2>&1
  ncu -i $out.ncu-rep --page source --csv --print-source sass > $out.sass.csv 2>/dev/null
  python tools/sass_hist.py $out.sass.csv 30 > $out.sass_hist.txt 2>&1
  ncu -i $out.ncu-rep --page raw --csv > $out.raw.csv 2>/dev/null
  gzip -f $out.src.csv $out.sass.csv; rm -f $out.ncu-rep
  cat $out.summary.txt; head -50 $out.lines.txt; head -34 $out.sass_hist.txt
done
