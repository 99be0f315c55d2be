# Round-end style GPU pass (box side): full GPU tests, smoke, default bench and the reference
# arm, then the ncu evidence round (launch lists + one --set full capture per hot kernel).
# usage: gpurun --timeout 5400 -- 'bash tools/gpu_round.sh r03'
TAG=${1:-rXX}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 3000 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 1500 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"
timeout 3000 bash tools/ncu_round.sh $TAG > gpurun_out/ncu_round.log 2>&1; echo "ncu round exit $?"
cat gpurun_out/bench.json
