# Round-end style GPU pass: full GPU tests, smoke, default bench, reference arm,
# launch list (cold, serialised) and one ncu --set full capture of K3.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-c4 --no-c5 > gpurun_out/ncu_bench.log 2>&1; echo "launches exit $?"
timeout 600 bash tools/ncu_capture.sh k3_full 'tc_contract_kernel' python tools/prof_c2.py 0.5 1; echo "k3 ncu exit $?"
timeout 600 bash tools/ncu_capture.sh k2_full 'recon_tile_kernel' python tools/prof_c2.py 0.5 1; echo "k2 ncu exit $?"
cat gpurun_out/bench.json
