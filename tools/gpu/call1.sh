set -x
nproc; free -g | head -2; lscpu | grep -E "Model name|Socket|Thread|Core" ; nvidia-smi --query-gpu=name,memory.total --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
NTFG_C5_PARITY_ITERS=5 timeout 2400 python -m pytest tests/test_config_parity_gpu.py -s -q --durations=0 -p no:cacheprovider 2>&1 | grep -v "^$" | tail -60
