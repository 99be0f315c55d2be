mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_tc_gpu.py -x -q -k "fast" > gpurun_out/pt_fast.log 2>&1; echo "pytest fast $?"; tail -15 gpurun_out/pt_fast.log
