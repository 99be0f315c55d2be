mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_unfold_gpu.py tests/test_cp_gpu.py tests/test_tucker_gpu.py tests/test_dropin_cpp.py -x -q > gpurun_out/pt_unf.log 2>&1; echo "pytest $?"; tail -25 gpurun_out/pt_unf.log
