mkdir -p gpurun_out
rm -f gpurun_out/trace_c5.txt gpurun_out/trace_c2.txt
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q > gpurun_out/pt_tc.log 2>&1; echo "pytest tc/cp $?"; tail -2 gpurun_out/pt_tc.log
NTFG_TC_TRACE=gpurun_out/trace_c5.txt timeout 300 python tools/prof_c5.py 256 1 > /dev/null 2>&1; python tools/tc_trace.py gpurun_out/trace_c5.txt 2>&1 | head -3
NTFG_TC_TRACE=gpurun_out/trace_c2.txt timeout 300 python tools/prof_c2.py 0.5 1 > /dev/null 2>&1; python tools/tc_trace.py gpurun_out/trace_c2.txt 2>&1 | head -3
timeout 300 python tools/bench_c5.py 2 1 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "c5 exit $?"; cat gpurun_out/c5.json
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench $?"
python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print({k:(v['ms_per_step']) for k,v in d['per_beta'].items()}, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['kernel_breakdown_ms_per_step'])"
