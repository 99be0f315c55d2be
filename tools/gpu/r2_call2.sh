./tools/mma_probe
timeout 600 python -m pytest tests/test_dropin_cpp.py tests/test_extrap_api.py -x -q -p no:cacheprovider 2>&1 | tail -5
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider --deselect tests/test_config_parity_gpu.py 2>&1 | tail -5
