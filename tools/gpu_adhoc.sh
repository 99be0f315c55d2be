mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_cli.py tests/test_dropin_cpp.py -x -q > gpurun_out/pt_cli.log 2>&1; echo "pytest cli $?"; tail -15 gpurun_out/pt_cli.log
