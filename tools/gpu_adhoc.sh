mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tc_gpu.py tests/test_cp_gpu.py -x -q > gpurun_out/pt_tc.log 2>&1; echo "pytest tc/cp $?"; tail -2 gpurun_out/pt_tc.log
timeout 300 python tools/bench_c5.py 2 1 > gpurun_out/c5.json 2> gpurun_out/c5.err; echo "c5 exit $?"; python -c "import json; d=json.load(open('gpurun_out/c5.json')); print(d['ms_per_step'], d['contract_avg_ms'], d['recon_ms'])"
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-c5 > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench $?"
python -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print({k:round(v['ms_per_step'],4) for k,v in d['per_beta'].items()}, d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['kernel_breakdown_ms_per_step'])"
