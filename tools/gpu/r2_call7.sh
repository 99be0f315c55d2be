timeout 600 python -m pytest tests/test_tc_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
rm -f /tmp/t.txt; NTFG_TC_TRACE=/tmp/t.txt timeout 600 python tools/prof_c5.py 1 | tail -1; python tools/tc_wstats.py /tmp/t.txt 5
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"recon_t" -c 2 python tools/prof_c5.py 1 2>&1 | grep -A3 "recon_tc_kernel" | grep -E "recon_tc|duration"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"recon_t" -c 2 python tools/prof_c2.py 0.5 1 2>&1 | grep -A3 "recon_tc_kernel" | grep -E "recon_tc|duration"
