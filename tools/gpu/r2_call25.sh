out=gpurun_out/prof_r02; name=c4_coo
timeout 900 ncu --set full --clock-control none --import-source on -k regex:coo_piece --launch-skip 4 -c 1 -o $out/$name python tools/prof_c4.py 2 > $out/$name.ncu.log 2>&1
python tools/ncu_summary.py $out/$name.ncu-rep > $out/$name.summary.txt 2>&1
ncu -i $out/$name.ncu-rep --page source --csv --print-source sass > $out/$name.sass.csv 2>/dev/null
python tools/sass_hist.py $out/$name.sass.csv 24 > $out/$name.sass_hist.txt 2>&1
ncu -i $out/$name.ncu-rep --page raw --csv > $out/$name.raw.csv 2>/dev/null
rm -f $out/$name.sass.csv $out/$name.ncu-rep
cat $out/$name.summary.txt
