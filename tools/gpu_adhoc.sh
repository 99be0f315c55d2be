mkdir -p gpurun_out
rm -f gpurun_out/trace_c5.txt gpurun_out/trace_c2.txt
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q > gpurun_out/pt_tc.log 2>&1; echo "pytest tc/cp $?"; tail -2 gpurun_out/pt_tc.log
NTFG_TC_TRACE=gpurun_out/trace_c5.txt timeout 300 python tools/prof_c5.py 256 1 > /dev/null 2>&1; python tools/tc_trace.py gpurun_out/trace_c5.txt 2>&1 | head -3
for mb in 1 2 3; do NTFG_TC_MBATCH=$mb timeout 300 python tools/bench_c5.py 2 1 > gpurun_out/c5_$mb.json 2> gpurun_out/c5.err; echo "c5 mb=$mb $(python -c "import json; d=json.load(open('gpurun_out/c5_$mb.json')); print(d['ms_per_step'], d['contract_avg_ms'], d['recon_ms'])")"; done
for mb in 1 2 3; do NTFG_TC_MBATCH=$mb timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-c5 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print('mb=$mb', {k:round(v['ms_per_step'],4) for k,v in d['per_beta'].items()}, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['kernel_breakdown_ms_per_step'])"; done
